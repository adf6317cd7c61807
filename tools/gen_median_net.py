#!/usr/bin/env python
"""Emit SVR_MED25_NET for svr_kernels.cuh: Batcher's odd-even merge sort on 32 wires, pruned to
the comparators whose outputs can reach wire 12.  With wires 25..31 held at +INF, wire 12 ends as
the 13th smallest of wires 0..24 (the pruned comparators never feed wire 12, so its value is the
full sorting network's).  Checked here against sorting on random inputs.

  python tools/gen_median_net.py > /tmp/net.h
"""
import random


def batcher(n):
    out, p = [], 1
    while p < n:
        k = p
        while k >= 1:
            j = k % p
            while j + k < n:
                for i in range(k):
                    if (i + j) // (2 * p) == (i + j + k) // (2 * p):
                        out.append((i + j, i + j + k))
                j += 2 * k
            k //= 2
        p *= 2
    return out


def pruned(target=12, wires=32):
    need, keep = {target}, []
    for a, b in reversed(batcher(wires)):
        if a in need or b in need:
            keep.append((a, b))
            need |= {a, b}
    return keep[::-1]


def main():
    net = pruned()
    rng = random.Random(1)
    for _ in range(20000):
        v = [rng.randint(-5, 300) for _ in range(25)] + [1 << 40] * 7
        for a, b in net:
            if v[a] > v[b]:
                v[a], v[b] = v[b], v[a]
        assert v[12] == sorted(v[:25])[12]
    body = " ".join("CE(%d, %d)" % p for p in net)
    print("// %d comparators (tools/gen_median_net.py)" % len(net))
    print("#define SVR_MED25_NET(CE) " + body)


if __name__ == "__main__":
    main()

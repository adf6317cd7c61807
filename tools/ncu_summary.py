#!/usr/bin/env python
"""Summarise an `ncu --set full` report into profiles/: one JSON line of key metrics per kernel
launch, plus the DRAM traffic of the insert kernel (feeds bench.py's roofline.traffic).

  python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r1_ncu_full_summary.jsonl \
      [--traffic profiles/insert_traffic.json --traffic-kernel k_pnn_lin]
"""
import argparse
import csv
import io
import json
import subprocess

KEYS = {
    "gpu__time_duration.sum": "duration",
    "smsp__inst_executed.sum": "warp_inst",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "launch__registers_per_thread": "regs",
    "launch__occupancy_limit_registers": "occ_limit_regs",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum": "smem_atom_bank_conflicts",
    "l1tex__t_requests_pipe_lsu_mem_global_op_red.sum": "global_red_requests",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio": "stall_long_sb",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio": "stall_wait",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio": "stall_barrier",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio": "stall_math_throttle",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio": "stall_lg_throttle",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum": "smem_atom_wavefronts",
    "lts__t_requests_srcunit_tex_op_red.sum": "l2_red_requests",
    "lts__t_sectors_srcunit_tex_op_red.sum": "l2_red_sectors",
    "lts__t_sectors_srcunit_tex_op_red_lookup_hit.sum": "l2_red_sectors_hit",
}


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True, check=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, units = r[0], r[1]
    for row in r[2:]:
        d = {"kernel": row[h.index("Kernel Name")].split("(")[0], "grid": row[h.index("Grid Size")],
             "block": row[h.index("Block Size")]}
        for k, name in KEYS.items():
            if k in h:
                v = row[h.index(k)].replace(",", "")
                try:
                    d[name] = float(v)
                except ValueError:
                    d[name] = v
                u = units[h.index(k)]
                if u:
                    d[name + "_unit"] = u
        yield d


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("out")
    ap.add_argument("--traffic")
    ap.add_argument("--traffic-kernel", default="k_pnn_lin")
    a = ap.parse_args()
    ds = list(rows(a.report))
    with open(a.out, "w") as f:
        for d in ds:
            f.write(json.dumps(d) + "\n")
    if a.traffic:
        ks = [d for d in ds if a.traffic_kernel in d["kernel"]]
        d = ks[0]
        with open(a.traffic, "w") as f:
            json.dump({"kernel": d["kernel"], "dram_bytes_per_launch": d["dram_read"] + d["dram_write"],
                       "smem_atom_wavefronts_per_launch": d.get("smem_atom_wavefronts"),
                       "l2_red_requests_per_launch": d.get("l2_red_requests"),
                       "l2_red_sectors_per_launch": d.get("l2_red_sectors"),
                       "l2_red_sector_hit_rate": (d["l2_red_sectors_hit"] / d["l2_red_sectors"])
                       if d.get("l2_red_sectors") else None,
                       "source": f"{a.out} (ncu --set full, cfg2 batch of 2400 frames, one launch)"},
                      f, indent=1)
    print(f"{len(ds)} launches summarised")


if __name__ == "__main__":
    main()

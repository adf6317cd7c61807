#!/usr/bin/env python
"""Insert-only timing of one BASELINE config via bench.measure_config (A/B helper).
usage: time_config.py NAME [STEPS]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

r = bench.measure_config(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 3)
print(json.dumps({k: r.get(k) for k in ("insert_ms", "value", "roofline_frac")}))

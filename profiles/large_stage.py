"""Run only the config-5-shaped stage workload of bench.py (MLP 4096-4096-4096-10,
bounds [0,2,3], iter_fisher, micro-batch 16) — a short target for ncu captures of
the kernels at HBM-bound sizes:

    ncu --set full -k regex:update_iter1 -s 20 -c 2 -o prof python profiles/large_stage.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

if __name__ == "__main__":
    import bench
    import paper_2503_12053_b200 as fb

    print(json.dumps(bench.large_stage_roofline(fb, 0), indent=1))

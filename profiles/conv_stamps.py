"""Summarise FERRET_CONV_STAMPS phase timestamps of the tensor-core conv kernel
(per CTA: start, setup done, first atom published, first MMA, last MMA committed,
accumulator ready, stores done) -> median phase durations per launch (us).

    FERRET_CONV_STAMPS=stamps.txt python profiles/conv_probe.py --tc 1 --modes 0
    python profiles/conv_stamps.py stamps.txt
"""
import sys

import numpy as np


def main(path):
    blocks, cur = [], None
    for line in open(path):
        if line.startswith("conv"):
            cur = [line.strip(), []]
            blocks.append(cur)
        elif cur is not None:
            cur[1].append([int(x) for x in line.split()])
    for head, rows in blocks:
        t = np.array(rows, dtype=np.float64)
        t = t[t[:, 0] > 0]
        t0 = t[:, 0].min()
        span = (t[:, 6].max() - t0) / 1e3
        med = lambda a, b: np.median(t[:, b] - t[:, a]) / 1e3
        print(f"{head}\n  span {span:6.1f} us  CTA start spread {(t[:, 0].max() - t0) / 1e3:5.1f} us | median: setup "
              f"{med(0, 1):5.2f} first-publish {med(1, 2):5.2f} first-mma {med(1, 3):5.2f} mma-span {med(3, 4):6.2f} "
              f"acc-ready {med(4, 5):5.2f} store {med(5, 6):5.2f} total {med(0, 6):6.2f}")


if __name__ == "__main__":
    main(sys.argv[1])

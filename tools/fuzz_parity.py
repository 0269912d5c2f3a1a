"""Randomised parity sweep (GPU vs the fp64 oracle) over geometries the test suite does not
enumerate: small and large batches (row groups / batch-as-M), narrow and wide channels, strides
1-4, filters 1-7, both dtypes, all three operators.  usage: python tools/fuzz_parity.py SEED COUNT
(test infrastructure: imports the oracle)."""
import os
import sys
import traceback

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
from cks_synth import Layer  # noqa: E402
from test_gpu_parity import check_full  # noqa: E402


def main():
    seed, count = int(sys.argv[1]), int(sys.argv[2])
    from paper_2306_15951_b200 import build
    build.build()
    rng = np.random.default_rng(seed)
    done = fails = 0
    while done < count:
        FH, FW = int(rng.choice([1, 2, 3, 4, 5, 7])), int(rng.choice([1, 2, 3, 4, 5, 7]))
        sh, sw = int(rng.integers(1, 5)), int(rng.integers(1, 5))
        ph, pw = int(rng.integers(0, FH)), int(rng.integers(0, FW))
        H, W = int(rng.integers(max(1, FH - 2 * ph), 48)), int(rng.integers(max(1, FW - 2 * pw), 40))
        C = int(rng.choice([1, 2, 3, 4, 8, 16, 32, 64, 96, 136]))
        OC = int(rng.choice([3, 8, 16, 32, 64, 96, 160, 264]))
        N = int(rng.choice([1, 2, 5, 16, 17, 31, 32, 33, 48, 64, 65, 100, 129]))
        dtype = "bf16" if rng.random() < 0.5 else "tf32"
        if dtype == "bf16" and C % 8 and rng.random() < 0.5:
            W = max(8, (W + 7) // 8 * 8)
        lay = Layer(f"fz{done}", N, C, H, W, OC, FH, FW, sh, sw, ph, pw)
        try:
            O.geom(**lay.geom())
        except O.GeometryError:
            continue
        if N * H * W * max(C, OC) > 3e6:
            continue
        done += 1
        try:
            check_full(torch, lay, dtype, config=21, idx=done)
        except Exception as e:  # report and continue
            fails += 1
            print("FAIL", dtype, lay, str(e)[:300], flush=True)
            traceback.print_exc(limit=2)
    print(f"fuzz seed {seed}: {done} geometries, {fails} failures", flush=True)


if __name__ == "__main__":
    main()

"""C5 inference micro-run for profiling: one 512^3 sample_volume of the
synthetic 2M-Gaussian field (bench.inference_c5 with reps=1)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402

if __name__ == "__main__":
    print(bench.inference_c5(reps=int(sys.argv[1]) if len(sys.argv) > 1 else 1))

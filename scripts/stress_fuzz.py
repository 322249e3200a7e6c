"""Race hunting: every fuzz case of tests/test_gpu_fuzz.py several times, each run
over a device heap pre-filled with garbage.  python scripts/stress_fuzz.py [reps] [first] [count]"""
import sys
import zlib  # noqa: F401
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import test_gpu_fuzz as T  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
first = int(sys.argv[2]) if len(sys.argv) > 2 else 0
count = int(sys.argv[3]) if len(sys.argv) > 3 else 160
bad = 0
for r in range(reps):
    for seed in range(first, first + count):
        junk = torch.full((int(5e8) // 4,), float(seed) + 0.25 + r, dtype=torch.float32, device="cuda")
        del junk
        try:
            T.test_fuzz_engine_vs_oracle(seed)
        except Exception as e:
            if type(e).__name__ == "Skipped":
                continue
            bad += 1
            print("FAIL rep", r, "seed", seed, type(e).__name__, str(e)[:100])
print(f"{reps} x seeds {first}..{first + count - 1}: {bad} failures")

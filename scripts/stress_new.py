"""Race hunting for the round-2c kernels: the cooperative tonal kernel (every ladder entry) and the
256x256 path with Nyquist-plane pairing, repeated over a device heap pre-filled with garbage.
    python scripts/stress_new.py [reps]"""
import os
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
os.environ["FM_RANGE_TAPS"] = "0"
import test_gpu_parity as P  # noqa: E402


class MP:
    def setenv(self, k, v):
        os.environ[k] = v


reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
bad = 0
for r in range(reps):
    for N in P.COOP_NS + [40, 162, 180]:
        junk = torch.full((int(5e8) // 4,), float(N) + 0.25 + r, dtype=torch.float32, device="cuda")
        del junk
        try:
            P.test_long_tonal_axes_every_ladder_entry(N, MP())
        except Exception as e:
            bad += 1
            print("FAIL coop rep", r, "N", N, type(e).__name__, str(e)[:100])
del os.environ["FM_RANGE_TAPS"]
for r in range(reps * 3):
    junk = torch.full((int(5e8) // 4,), 0.5 + r, dtype=torch.float32, device="cuda")
    del junk
    try:
        P.test_wide_se_big_tiles()
    except Exception as e:
        bad += 1
        print("FAIL big rep", r, type(e).__name__, str(e)[:100])
print(f"stress_new: {bad} failures")
sys.exit(1 if bad else 0)

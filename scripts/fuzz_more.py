"""Extended GPU fuzz: the randomized engine-vs-C-oracle cases of tests/test_gpu_fuzz.py
over a further seed range (the test suite runs seeds 0..159).

    python scripts/fuzz_more.py [first_seed] [count]
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import test_gpu_fuzz as T  # noqa: E402

first = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
count = int(sys.argv[2]) if len(sys.argv) > 2 else 600
bad = skipped = 0
for seed in range(first, first + count):
    try:
        T.test_fuzz_engine_vs_oracle(seed)
    except AssertionError as e:
        bad += 1
        print("FAIL", seed, e)
    except Exception as e:  # pytest.skip raises Skipped
        if type(e).__name__ == "Skipped":
            skipped += 1
        else:
            bad += 1
            print("ERR", seed, type(e).__name__, e)
print(f"seeds {first}..{first + count - 1}: failures {bad}, skipped {skipped}")
sys.exit(1 if bad else 0)

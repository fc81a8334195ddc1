"""Find the first fuzz program whose co-executed B200 run differs from the imperative oracle (debug aid)."""
import sys, traceback
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from programs import fuzz_program
from oracle.cpu_backend import CpuBackend
from paper_2201_09210_b200.b200 import B200Backend
from test_gpu_coexec import run, assert_close
first = int(sys.argv[1]) if len(sys.argv) > 1 else 0
last = int(sys.argv[2]) if len(sys.argv) > 2 else 200
for seed in range(first, last):
    src = fuzz_program(seed)
    ref, _, _ = run(src, "imperative", CpuBackend())
    be = B200Backend(precision="f64")
    try:
        got, st, _ = run(src, "coexec", be)
        assert_close(ref, got, 1e-12, "sigmoid" not in src)
    except Exception as e:
        print("SEED", seed, type(e).__name__, str(e)[:300])
        print(src)
        traceback.print_exc(limit=3)
        break
    finally:
        try: be.close()
        except Exception: pass

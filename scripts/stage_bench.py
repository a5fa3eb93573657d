"""Per-stage times (bench.py step, CUDA events, L2 flushed) of several builds of
the library on one workload, each in its own process.
usage: python scripts/stage_bench.py workload lib1.so lib2.so ..."""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
w = sys.argv[1]
for lib in sys.argv[2:]:
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--workload", w, "--steps", "10",
                          "--warmup", "3", "--no-cpu-baseline", "--no-e2e", "--no-dense", "--no-f1"],
                         env=dict(os.environ, SPARGE_LIB=lib), capture_output=True, text=True).stdout
    d = json.loads(out.strip().splitlines()[-1])
    print(f"{lib:45s} {w:16s} " + " ".join(f"{k} {v:.4f}" for k, v in d["stages_ms"].items()), flush=True)

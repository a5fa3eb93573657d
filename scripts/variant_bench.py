"""Time k_sparse_attn alone (CUDA events, L2 flushed) for several builds of
the library (SPARGE_LIB=...), on one workload.  Each variant runs in its own
process.  usage: python scripts/variant_bench.py workload lib1.so lib2.so ..."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, ROOT)
    import numpy as np, torch
    import bench
    from paper_2502_18137_b200 import inputs, sparge
    w = sys.argv[2]
    cfg = bench.workload_cfg(w)
    q, k, v = (inputs.to_device(a) for a in bench.gen_inputs(cfg, 1000))
    perm_np = bench.hilbert_perm(cfg)
    perm = None if perm_np is None else torch.from_numpy(perm_np).cuda()
    o, bf = sparge.sparge_forward(q, k, v, cfg["tau"], cfg["theta"], cfg["lam"], causal=cfg["causal"], perm=perm)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for it in range(13):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        sparge.sparge_attn_fwd_ex(bf.shape, bf.qq, bf.dq, bf.kq, bf.dk, v, bf.lut, bf.cnt, cfg["lam"], perm, o,
                                  None, bf.workspace, sparge.SPARGE_ATTN_SKIP_VPREP)
        b.record(); torch.cuda.synchronize()
        if it >= 3: ts.append(a.elapsed_time(b))
    print(f"{os.environ['SPARGE_LIB']:45s} {w:16s} attn {np.median(ts):.4f} ms (min {min(ts):.4f})", flush=True)
    sys.exit(0)
w = sys.argv[1]
for lib in sys.argv[2:]:
    subprocess.run([sys.executable, os.path.abspath(__file__), "--child", w], env=dict(os.environ, SPARGE_LIB=lib))

"""Per-CTA timeline of k_sparse_attn (debug build -DSPARGE_CTA_TIMING):
where does the attention time go between the softmax loop and the rest
(launch gaps, prologue, epilogue, tail)?  GPU only.
usage: python scripts/cta_timeline.py [workload]"""
import ctypes, os, sys
os.environ["SPARGE_LIB"] = "libsparge_sparge_cta_timing.so"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2502_18137_b200 import inputs, sparge
w = sys.argv[1] if len(sys.argv) > 1 else "llama31_8b_32k"
cfg = bench.workload_cfg(w)
q, k, v = (inputs.to_device(a) for a in bench.gen_inputs(cfg, 1000))
perm_np = bench.hilbert_perm(cfg)
perm = None if perm_np is None else torch.from_numpy(perm_np).cuda()
o, bf = sparge.sparge_forward(q, k, v, cfg["tau"], cfg["theta"], cfg["lam"], causal=cfg["causal"], perm=perm)
torch.cuda.synchronize()
for _ in range(2):
    sparge.sparge_attn_fwd_ex(bf.shape, bf.qq, bf.dq, bf.kq, bf.dk, v, bf.lut, bf.cnt, cfg["lam"], perm, o,
                              None, bf.workspace, sparge.SPARGE_ATTN_SKIP_VPREP)
torch.cuda.synchronize()
lib = ctypes.CDLL(sparge.LIB_PATH)
n = bf.shape.B * bf.shape.Hq * ((bf.shape.N + 127) // 128)
rec = np.zeros((1 << 16, 6), np.uint64)
assert lib.sparge_debug_cta_records(rec.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(rec.nbytes)) == 0
r = rec[:n].astype(np.int64)
if os.environ.get("CTA_DUMP"):
    np.save(os.environ["CTA_DUMP"], r)
t0 = r[:, 0].min()
entry, lstart, lend, exit_, sm, nt = (r[:, i] for i in range(6))
span = exit_.max() - t0
print(f"{w}: {n} CTAs, kernel span {span/1e3:.1f} us")
print(f"  per CTA mean: prologue (entry->loop) {np.mean(lstart-entry)/1e3:.2f} us, loop {np.mean(lend-lstart)/1e3:.2f} us, "
      f"epilogue (loop end->exit) {np.mean(exit_-lend)/1e3:.2f} us, tiles {nt.mean():.1f}")
print(f"  loop ns per tile (sum loop / sum tiles): {np.sum(lend-lstart)/max(1,nt.sum()):.0f}")
# per SM: busy time and gaps between consecutive CTAs
busy = []; gaps = []
for s in np.unique(sm):
    idx = np.where(sm == s)[0]
    order = idx[np.argsort(entry[idx])]
    e, x = entry[order], exit_[order]
    busy.append(np.sum(x - e))
    # two CTAs resident: a new CTA starts when one exits
    ends = np.sort(x)
    gaps.append(np.sum(np.maximum(0, e[2:] - ends[:len(e) - 2])))
print(f"  SMs {len(busy)}; mean SM CTA-busy {np.mean(busy)/1e3:.1f} us (2 slots -> slot-time {np.mean(busy)/2e3:.1f} us of span {span/1e3:.1f})")
starts = [entry[sm == s].min() - t0 for s in np.unique(sm)]
fins = [exit_.max() - exit_[sm == s].max() for s in np.unique(sm)]
print(f"  per SM: slot gaps between CTAs {np.mean(gaps)/2e3:.1f} us per slot, "
      f"first entry after kernel start {np.mean(starts)/1e3:.1f} us, idle after its last CTA {np.mean(fins)/1e3:.1f} us")
print(f"  last CTA exit minus median SM finish: {(exit_.max() - np.median([exit_[sm==s].max() for s in np.unique(sm)]))/1e3:.1f} us")

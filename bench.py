#!/usr/bin/env python
"""SpargeAttn hot-path benchmark (contract: DESIGN.md §7).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME] [--impl reference]

One step = the whole hot path on one batch element of the
workload: a1 quantise Q and K (+ pool + CosSim), a2 predict the block mask,
a3 stage V^T and run the sparse attention kernel.  The metric is the paper's
speed 1/t = O(attn)/t in TOPS, with O(attn) the dense attention op
count (4 N^2 d H, causal: 4 d H N(N+1)/2, reading R8-v) and t the device time
of the step (prediction included).

Multi-GPU (torchrun): the heads of ONE sequence are split by
contiguous kv-groups across ranks (--shard heads, default), each rank
generating its shard from per-global-head seeds -- no data-path collective;
value = the whole job's dense ops / max-over-ranks step time ("scaling":
"strong").  After timing, O is all-gathered over NCCL and compared bit for
bit with one GPU running every head.  --shard batch gives every rank its own
sequence instead (weak scaling).

Hyper-parameters: each workload runs at the triple the §3.6 tuner found at
the paper's accuracy bounds (inputs.TUNED <- profiles/r02_f2_tuned.json,
P:L469); --triple fixed selects round 1's tau=.9/theta=.5/lambda=-5 (R20).
The default line also carries the configs[4] sweep (8K..128K, each point at
its own tuned triple).  Inputs are synthetic (paper_2502_18137_b200.inputs);
the oracle (oracle/) is used only for the cpu_baseline leg, the parity
figures and --impl reference.
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "effective attention TOPS & sparsity at seq 8K–128K vs dense; L1 err vs oracle"
LOG2E = 1.4426950408889634


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="llama31_8b_32k")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-f1", action="store_true",
                    help="skip the NEXT-row variants (f1 bf16 QK, f4 FP8 PV)")
    ap.add_argument("--profile", action="store_true",
                    help="minimal run for ncu: warmup + steps only, no side legs")
    ap.add_argument("--out", default=None, help="also write the JSON line here")
    ap.add_argument("--tau", type=float, default=None, help="override tau")
    ap.add_argument("--theta", type=float, default=None, help="override theta")
    ap.add_argument("--lam", type=float, default=None, help="override lambda")
    ap.add_argument("--triple", default="tuned", choices=["tuned", "fixed"],
                    help="tuned: inputs.TUNED (the §3.6 tuner at the paper's bounds); "
                         "fixed: tau=.9 theta=.5 lambda=-5 (R20)")
    ap.add_argument("--shard", default="heads", choices=["heads", "batch"],
                    help="multi-GPU partition (SURVEY §8(e)): kv-groups of one sequence, "
                         "or one sequence per rank")
    ap.add_argument("--no-sweep", action="store_true", help="skip the 8K..128K sweep leg")
    ap.add_argument("--no-gather-check", action="store_true")
    return ap.parse_args()


# ------------------------------------------------------------------ workload
def workload_cfg(name):
    from paper_2502_18137_b200 import inputs
    cfg = dict(inputs.WORKLOADS[name])
    cfg.update(inputs.HYPER)
    cfg["triple"] = "fixed (R20)"
    if cfg["kind"] == "video":
        cfg["N"] = cfg["text_prefix"] + cfg["T"] * cfg["H"] * cfg["W"]
    return cfg


def gen_inputs(cfg, seed, heads=None):
    """float32 numpy [1, H, N, d] arrays + optional Hilbert perm (numpy int32)."""
    from paper_2502_18137_b200 import inputs
    perm = None
    if cfg["kind"] in ("llm_local", "llm_rope"):
        gen = inputs.llm_rope if cfg["kind"] == "llm_rope" else inputs.llm_local
        q, k, v = gen(seed, cfg["N"], d=cfg["d"], Hq=cfg["Hq"], Hkv=cfg["Hkv"], heads=heads)
    elif cfg["kind"] == "video":
        q, k, v = inputs.video(seed, cfg["T"], cfg["H"], cfg["W"], d=cfg["d"], heads=cfg["Hq"],
                               text_prefix=cfg["text_prefix"], heads_subset=heads)
    else:
        q, k, v = inputs.planted(seed, N=cfg["N"], d=cfg["d"], heads=cfg["Hq"])
    return q, k, v


def hilbert_perm(cfg):
    if not cfg.get("hilbert"):
        return None
    from paper_2502_18137_b200 import sparge
    perm, _ = sparge.hilbert_permute(cfg["T"], cfg["H"], cfg["W"], cfg["text_prefix"])
    return perm


def dense_ops(cfg, B=1):
    N, d, H = cfg["N"], cfg["d"], cfg["Hq"]
    if cfg["causal"]:
        return 4.0 * d * H * B * N * (N + 1) / 2.0
    return 4.0 * d * H * B * N * N


def sample_qblocks(tm, seed=0, n=8):
    """The first, second, middle and last query blocks plus random ones, n in all."""
    rng = np.random.default_rng(seed)
    base = {b for b in (0, 1, tm // 2, tm - 1) if 0 <= b < tm}
    rest = [b for b in rng.permutation(tm).tolist() if b not in base]
    return sorted(base.union(rest[:max(0, min(n, tm) - len(base))]))


def sample_dense_ops(cfg, qblocks):
    N, d = cfg["N"], cfg["d"]
    ops = 0.0
    for i in qblocks:
        for r in range(i * 128, min((i + 1) * 128, N)):
            ops += 4.0 * d * ((r + 1) if cfg["causal"] else N)
    return ops


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md)."""
    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_id):
        self.gpu_id = gpu_id
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu_id), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.2)
        except OSError:
            self.proc = None
        self.t0 = time.time()          # the timed region starts now
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        self.t1 = time.time()          # ... and ended (after the synchronize)
        if self.proc:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        import datetime
        outside = 0
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                if not (self.t0 - 0.05 <= ts <= self.t1 + 0.05):   # one 50-ms sample of slack
                    outside += 1
                    continue
            except (ValueError, AttributeError):
                pass
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0,
                    "note": f"no 50-ms nvidia-smi sample fell inside the "
                            f"{1e3 * (self.t1 - self.t0):.0f}-ms timed region ({outside} outside it)"}
        busy = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(busy), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}

# ------------------------------------------------------------------ our arm
STAGES = ["quant_ms", "predict_ms", "vprep_ms", "attn_ms"]
# kernels per step: quantise Q, quantise K, S^ DMMA, TopCdf rows, V^T stage,
# launch order x2, attention
LAUNCHES_PER_STEP = 8


class Problem:
    """One rank's share of a workload on its GPU: inputs resident in HBM
    (plus pinned host copies for the e2e leg), the C-ABI shape and buffers.

    shard="heads" (multi-GPU default): contiguous kv-groups of
    ONE sequence per rank, generated from per-global-head seeds, so nothing
    is sent; shard="batch": every rank its own sequence (seed 1000 + rank)."""

    def __init__(self, cfg, world, rank, dev, shard="heads", seed=1000, pin=True):
        import torch
        from paper_2502_18137_b200 import inputs, multigpu, sparge
        self.cfg, self.dev = cfg, dev
        N, d, Hq, Hkv = cfg["N"], cfg["d"], cfg["Hq"], cfg["Hkv"]
        if shard == "heads" and world > 1:
            self.hq, self.hkv = multigpu.local_heads(Hq, Hkv, world, rank)
            heads = self.hq
        else:
            self.hq, self.hkv = list(range(Hq)), list(range(Hkv))
            heads = None
            if shard == "batch":
                seed = seed + rank
        self.shard, self.world = shard, world
        self.Hq, self.Hkv = len(self.hq), len(self.hkv)
        self.empty = self.Hq == 0
        self.perm_np = hilbert_perm(cfg)
        self.perm = None if self.perm_np is None else torch.from_numpy(self.perm_np).to(dev)
        if self.empty:
            return
        qn, kn, vn = gen_inputs(cfg, seed=seed, heads=heads)
        self.host = tuple(inputs.to_device(a, device="cpu", pin=pin) for a in (qn, kn, vn))
        del qn, kn, vn
        self.q, self.k, self.v = (t.to(dev) for t in self.host)
        self.shape = sparge.make_shape(1, self.Hq, self.Hkv, N, d, cfg["causal"], self.q.dtype)
        self.bf = sparge.Buffers(self.shape, device=dev)
        self.o = torch.empty_like(self.q)
        tm, tn = math.ceil(N / 128), math.ceil(N / 64)
        if cfg["causal"]:
            self.live = sum(min(tn, (min((i + 1) * 128, N) - 1) // 64 + 1)
                            for i in range(tm)) * self.Hq
        else:
            self.live = tm * tn * self.Hq

    def ops(self):
        """Dense attention ops of this rank's share (R8-v)."""
        c = dict(self.cfg)
        c["Hq"] = self.Hq
        return dense_ops(c)

    def step(self, ev=None, counters=None, tau=None, theta=None, lam=None, shape=None, bf=None,
             o=None):
        """One pass of the whole hot path: a1(Q), a1(K), a2, V stage, a3."""
        from paper_2502_18137_b200 import sparge
        if self.empty:
            for e in (ev or []):
                e.record()
            return
        cfg = self.cfg
        tau = cfg["tau"] if tau is None else tau
        theta = cfg["theta"] if theta is None else theta
        lam = cfg["lam"] if lam is None else lam
        shape = self.shape if shape is None else shape
        bf = self.bf if bf is None else bf
        o = self.o if o is None else o
        q, k, v, perm = self.q, self.k, self.v, self.perm
        if ev: ev[0].record()
        sparge.sparge_quantize(shape, q, 0, perm, bf.qq, bf.dq, bf.q_pooled, bf.q_sim)
        if shape.smooth_k:        # row f4 K smoothing: mean, then INT8 of K - mean
            sparge.sparge_smooth_k_mean(shape, k, bf.smooth_workspace, bf.k_mean)
            sparge.sparge_quantize_smooth_k(shape, k, perm, bf.k_mean, bf.kq, bf.dk, bf.k_pooled,
                                            bf.k_sim)
        else:
            sparge.sparge_quantize(shape, k, 1, perm, bf.kq, bf.dk, bf.k_pooled, bf.k_sim)
        if ev: ev[1].record()
        sparge.sparge_predict_mask(shape, bf.q_pooled, bf.q_sim, bf.k_pooled, bf.k_sim, tau, theta,
                                   bf.mask, bf.lut, bf.cnt, bf.pred_workspace)
        if not ev:
            # one attention call: k_order, the V stage overlapping it, the
            # attention kernel (the product path, sparge_forward's call)
            sparge.sparge_attn_fwd(shape, bf.qq, bf.dq, bf.kq, bf.dk, v, bf.lut, bf.cnt, lam,
                                   perm, o, counters, bf.workspace)
            return
        ev[2].record()
        sparge.sparge_attn_fwd_ex(shape, bf.qq, bf.dq, bf.kq, bf.dk, v, bf.lut, bf.cnt, lam, perm,
                                  o, counters, bf.workspace, sparge.SPARGE_ATTN_VPREP_ONLY)
        ev[3].record()
        sparge.sparge_attn_fwd_ex(shape, bf.qq, bf.dq, bf.kq, bf.dk, v, bf.lut, bf.cnt, lam, perm,
                                  o, counters, bf.workspace, sparge.SPARGE_ATTN_SKIP_VPREP)
        ev[4].record()

    def dense_reference(self):
        """Full attention without quantisation or sparsity: the f1 kernel with
        tau = 1, theta = -1, lambda = -inf (bf16 QK^T, fp32 softmax; the
        tuner's reference O', reading R25)."""
        import torch
        from paper_2502_18137_b200 import sparge
        ref = torch.empty_like(self.q)
        sparge.sparge_forward(self.q, self.k, self.v, 1.0, -1.0, -math.inf,
                              causal=self.cfg["causal"], perm=self.perm, out=ref,
                              qk_dtype=sparge.SPARGE_QK_INPUT, counters=False)
        return ref


def all_sum(vals, dev):
    """Sum host numbers over ranks (counters / L1 sums)."""
    import torch
    import torch.distributed as dist
    if dist.is_initialized() and dist.get_backend() == "gloo":
        dev = "cpu"
    t = torch.tensor([float(x) for x in vals], dtype=torch.float64, device=dev)
    if dist.is_initialized():
        dist.all_reduce(t)
    return t.tolist()


def time_steps(prob, K, W, flush, sync, clock=False, **kw):
    """W untimed warm-up steps, then K steps with L2 flushed between them,
    each bracketed by two CUDA events on the launching stream and NOTHING in
    between (an event record between two kernels would end the programmatic
    dependent launch overlap of the step's kernels, sparge_internal.h), then
    min(K, 10) more steps with an event between stages for the breakdown.
    Returns (per-step ms [K], per-stage ms [min(K,10), 4], clock summary or
    None)."""
    import torch
    for _ in range(W):
        prob.step(**kw)
    torch.cuda.synchronize()
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    sync()
    torch.cuda.synchronize()
    clk = None
    if clock:
        props = torch.cuda.get_device_properties(prob.dev)
        gpu_id = str(props.uuid)
        gpu_id = gpu_id if gpu_id.startswith("GPU-") else f"GPU-{gpu_id}"
        clk = ClockSampler(gpu_id)
        clk.__enter__()
    for s in range(K):
        flush.zero_()                          # L2 flush between steps (not timed)
        ev0[s].record()
        prob.step(**kw)
        ev1[s].record()
    torch.cuda.synchronize()
    if clk is not None:
        clk.__exit__(None, None, None)
    sync()
    tot = np.array([ev0[s].elapsed_time(ev1[s]) for s in range(K)])
    S = min(K, 10)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(S)]
    for s in range(S):
        flush.zero_()
        prob.step(ev=evs[s], **kw)
    torch.cuda.synchronize()
    st = np.array([[evs[s][a].elapsed_time(evs[s][a + 1]) for a in range(4)] for s in range(S)])
    return tot, st, (clk.summary() if clk is not None else None)


def counters_of(prob, dev):
    """(qk tiles, PV warp slices, PV MMAs, live tiles) summed over ranks."""
    if prob.empty:
        return all_sum([0, 0, 0, 0], dev)
    c = prob.bf.counters.cpu().numpy().astype(np.int64)
    return all_sum([c[0, :, 0].sum(), c[0, :, 1].sum(), c[0, :, 2].sum(), prob.live], dev)


def l1_vs_dense(prob, dev):
    """Relative L1 of this step's O against full attention (R25), whole job."""
    from paper_2502_18137_b200 import sparge
    if prob.empty:
        return all_sum([0.0, 0.0], dev)
    ref = prob.dense_reference()
    s = sparge.sparge_l1_sums(prob.o, ref)[:2].cpu().tolist()
    del ref
    return all_sum(s, dev)


def sparsity_from(c):
    qk, pv, _, live = c
    return 1.0 - (qk + pv / 4.0) / (2.0 * live) if live else 0.0


def roofline_of(d, qk_exec, pv_slices, attn_ms, workload):
    per_tile_qk = 2.0 * 128 * 64 * d
    per_slice_pv = 2.0 * 32 * 64 * d
    ops_qk = qk_exec * per_tile_qk
    ops_pv = pv_slices * per_slice_pv
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        bf16_peak, peak_src = float(peaks["bf16_tflops"]), "measured"
    except Exception:
        bf16_peak, peak_src = 1590.0, "fallback"
    i8_peak = 2.0 * bf16_peak          # INT8 dense = 2x bf16 (nominal ratio, 4.5 vs 2.25 POPS)
    tot = ops_qk + ops_pv
    mix_peak = tot / (ops_qk / i8_peak + ops_pv / bf16_peak) if tot else i8_peak
    sheet_peak = tot / (ops_qk / 4500.0 + ops_pv / 2250.0) if tot else 4500.0
    achieved = tot / (attn_ms * 1e-3) / 1e12 if attn_ms > 0 else 0.0
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "attn_traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get(workload)
    return {"bound": "tensor", "kernel": "k_sparse_attn", "achieved": achieved,
            "peak": mix_peak, "unit": "TFLOP/s", "frac": achieved / mix_peak,
            "traffic": traffic,
            "frac_datasheet": achieved / sheet_peak,
            "peak_note": f"INT8 QK at 2x bf16 {peak_src} ({i8_peak:.0f}) + bf16 PV "
                         f"({bf16_peak:.0f}), weighted by the executed op mix; frac_datasheet "
                         f"uses the nominal 4500/2250 TOPS mix ({sheet_peak:.0f})"}, bf16_peak


def mufu_roofline_of(qk_exec, attn_ms, n_sm, clk_mhz):
    """The attention kernel's second bound: every kept 128x64 tile
    exponentiates its 8192 entries on the MUFU (ex2.approx, 16 per clock per
    SM: scripts/ubench_mufu_*.cu), so exp2/s against 16 x SMs x the maximum
    SM clock is the fraction of that pipe's peak."""
    exps = qk_exec * 128.0 * 64.0
    achieved = exps / (attn_ms * 1e-3) / 1e9 if attn_ms > 0 else 0.0
    peak = 16.0 * n_sm * clk_mhz * 1e6 / 1e9
    return {"bound": "mufu", "kernel": "k_sparse_attn", "achieved": achieved, "peak": peak,
            "unit": "Gexp2/s", "frac": achieved / peak if peak else None,
            "note": f"8192 ex2 per executed QK tile; peak = 16/clk/SM x {n_sm} SMs x {clk_mhz:.0f} MHz"}


def hyper(cfg, name, triple):
    """tau/theta/lambda of a workload: the §3.6 tuner's values at the paper's
    bounds (inputs.TUNED, profiles/r02_f2_tuned.json) or the fixed R20 triple."""
    from paper_2502_18137_b200 import inputs
    if triple == "tuned" and name in inputs.TUNED:
        t = inputs.TUNED[name]
        cfg.update(tau=t["tau"], theta=t["theta"], lam=t["lambda"], triple="tuned",
                   l1_bound=t["l1_bound"])
    else:
        cfg.update(inputs.HYPER)
        cfg["triple"] = "fixed (R20)"
    return cfg


def measure_workload(name, args, world, rank, dev, flush, sync, K, W, dense=True):
    """One workload at its own triple: TOPS, sparsity, stages, L1 vs dense,
    dense comparator (used by the sweep leg)."""
    import torch
    from paper_2502_18137_b200 import multigpu
    cfg = hyper(workload_cfg(name), name, args.triple)
    prob = Problem(cfg, world, rank, dev, args.shard, pin=False)
    if not prob.empty:
        prob.bf.counters.zero_()
        prob.step(counters=prob.bf.counters)
    c = counters_of(prob, dev)
    tot, st, _ = time_steps(prob, K, W, flush, sync)
    ms = multigpu.max_over_ranks(float(tot.mean()), dev)
    ops_total = dense_ops(cfg) * (world if args.shard == "batch" else 1)
    s1, s2 = l1_vs_dense(prob, dev)
    stages = dict(zip(STAGES, st.mean(0).tolist()))
    out = {"workload": name, "N": cfg["N"], "tau": cfg["tau"], "theta": cfg["theta"],
           "lambda": cfg["lam"], "triple": cfg["triple"], "value": ops_total / (ms * 1e-3) / 1e12,
           "unit": "TOPS", "ms_per_step": ms, "sparsity": sparsity_from(c), "stages_ms": stages,
           "predict_over_attn": stages["predict_ms"] / stages["attn_ms"] if stages["attn_ms"] else None,
           "l1_vs_dense": s1 / s2 if s2 else None}
    if dense:
        Kd = max(2, min(K, 5))
        totd, std, _ = time_steps(prob, Kd, 1, flush, sync, tau=1.0, theta=-1.0, lam=-math.inf)
        dms = multigpu.max_over_ranks(float(totd.mean()), dev)
        out["dense_value"] = ops_total / (dms * 1e-3) / 1e12
        # Table 3's overhead: prediction time over the FULL
        # (dense) attention time -- the dense comparator's attention stage
        dattn = float(std[:, 3].mean())
        out["dense_attn_ms"] = dattn
        out["predict_over_dense_attn"] = stages["predict_ms"] / dattn if dattn else None
        out["speedup"] = out["value"] / out["dense_value"]
        out["target_0.8/(1-s)"] = 0.8 / max(1e-9, 1.0 - out["sparsity"])
    del prob
    torch.cuda.empty_cache()
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2502_18137_b200 import multigpu, shard, sparge

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # SPARGE_BENCH_ONE_GPU=1 (plumbing checks on a 1-GPU box only: every rank
    # on cuda:0, gloo instead of NCCL -- timings are then meaningless)
    one_gpu = os.environ.get("SPARGE_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)        # before NCCL init: one GPU per rank
    dev = torch.device("cuda", local)
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    cfg = hyper(workload_cfg(args.workload), args.workload, args.triple)
    for key in ("tau", "theta", "lam"):
        if getattr(args, key) is not None:
            cfg[key] = getattr(args, key)
            cfg["triple"] = "override"
    N, d, Hq, Hkv = cfg["N"], cfg["d"], cfg["Hq"], cfg["Hkv"]

    def sync():
        if world > 1:
            dist.barrier()

    t_perm = time.perf_counter()
    prob = Problem(cfg, world, rank, dev, args.shard)
    perm_host_ms = 1e3 * (time.perf_counter() - t_perm) if prob.perm_np is not None else 0.0
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)

    # one untimed step for sparsity / counters / parity samples
    if not prob.empty:
        prob.bf.counters.zero_()
        prob.step(counters=prob.bf.counters)
        sparge.sparge_attn_status(prob.bf.workspace)
    c = counters_of(prob, dev)
    qk_exec, pv_slices, pv_mma, live = (int(x) for x in c)
    sparsity = sparsity_from(c)
    snap = None
    if rank == 0 and not prob.empty:
        snap = (prob.o[0, 0].float().cpu(), prob.bf.mask[0, 0].cpu())   # head 0 for the parity leg

    K, W = args.steps, args.warmup
    tot, st, clk = time_steps(prob, K, W, flush, sync, clock=True)
    ms = multigpu.max_over_ranks(float(tot.mean()), dev)
    stages = dict(zip(STAGES, st.mean(0).tolist()))
    ops_total = dense_ops(cfg) * (world if args.shard == "batch" else 1)
    value = ops_total / (ms * 1e-3) / 1e12
    # the dominant kernel on this rank (rank 0's share; its own counters)
    c_loc = prob.bf.counters.cpu().numpy().astype(np.int64) if not prob.empty else np.zeros((1, 1, 3))
    roofline, bf16_peak = roofline_of(d, int(c_loc[0, :, 0].sum()), int(c_loc[0, :, 1].sum()),
                                      stages["attn_ms"], args.workload)
    try:
        sm_max = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["sm_max_mhz"])
    except Exception:
        sm_max = 1965.0
    roofline_mufu = mufu_roofline_of(int(c_loc[0, :, 0].sum()), stages["attn_ms"],
                                     torch.cuda.get_device_properties(dev).multi_processor_count,
                                     sm_max)
    if world > 1 and args.shard == "heads":
        par = f"heads: kv-groups split over {world} ranks (no data-path collective)"
    elif world > 1:
        par = f"batch x{world} (independent sequences, no collective)"
    else:
        par = "single GPU"
    result = {
        "metric": METRIC, "value": value, "unit": "TOPS", "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak" if (world > 1 and args.shard == "batch") else "strong",
        "vs_baseline": None, "dtype": "int8+bf16", "data": "synthetic",
        "config": {"workload": args.workload, "B": world if args.shard == "batch" else 1,
                   "N": N, "d": d, "Hq": Hq, "Hkv": Hkv, "causal": bool(cfg["causal"]),
                   "hilbert": bool(cfg.get("hilbert")), "tau": cfg["tau"],
                   "theta": cfg["theta"], "lambda": cfg["lam"], "triple": cfg["triple"],
                   "parallelism": par, "heads_per_rank": prob.Hq,
                   "l2": "flushed (512 MB write) between timed steps"},
        "sparsity": sparsity,
        "counters": {"qk_tiles": qk_exec, "pv_warp_slices": pv_slices, "pv_mmas": pv_mma,
                     "live_tiles": live},
        "stages_ms": stages,
        "predict_over_attn": stages["predict_ms"] / stages["attn_ms"] if stages["attn_ms"] else None,
        "permutation": {"hilbert": prob.perm_np is not None, "host_build_ms": perm_host_ms,
                        "note": "a0 index build on the host once per shape; the gather is "
                                "fused into a1 / the V stage and the scatter into a3"},
        "roofline": roofline,
        "roofline_mufu": roofline_mufu,
        "gpu_launches": (0 if prob.empty else LAUNCHES_PER_STEP) * K,
        "clocks": clk,
    }
    if world > 1:
        result["multi_gpu"] = {"partition": args.shard, "static_efficiency":
                               shard.static_efficiency(Hkv, world) if args.shard == "heads" else 1.0}
    if args.profile:
        emit(result, rank, args)
        return

    # ---- accuracy at this triple: L1 vs full attention, whole job ----
    s1, s2 = l1_vs_dense(prob, dev)
    result["accuracy"] = {"l1_vs_dense": s1 / s2 if s2 else None,
                          "l1_bound_paper": cfg.get("l1_bound"),
                          "reference": "full attention, no quantisation or sparsity (the f1 "
                                       "kernel, tau=1 theta=-1 lambda=-inf; R25)"}

    # ---- dense comparator: same kernels, all-ones mask, lambda = -inf ----
    if not args.no_dense:
        totd, std, _ = time_steps(prob, min(K, 10), 1, flush, sync, tau=1.0, theta=-1.0,
                                  lam=-math.inf)
        dms = multigpu.max_over_ranks(float(totd.mean()), dev)
        dense_value = ops_total / (dms * 1e-3) / 1e12
        dattn = float(std[:, 3].mean())
        result["dense"] = {"value": dense_value, "ms_per_step": dms,
                           "attn_ms": dattn,
                           "speedup": value / dense_value,
                           "target_0.8/(1-s)": 0.8 / max(1e-9, 1.0 - sparsity)}
        # Table 3's overhead: prediction over FULL attention
        result["predict_over_dense_attn"] = stages["predict_ms"] / dattn if dattn else None

    # ---- the fixed R20 triple on the same inputs (round 1's headline) ----
    if args.triple == "tuned" and not prob.empty:
        from paper_2502_18137_b200 import inputs as _in
        fx = _in.HYPER
        prob.bf.counters.zero_()
        prob.step(counters=prob.bf.counters, tau=fx["tau"], theta=fx["theta"], lam=fx["lam"])
        cf = counters_of(prob, dev)
        totf, stf, _ = time_steps(prob, min(K, 10), 2, flush, sync, tau=fx["tau"],
                                  theta=fx["theta"], lam=fx["lam"])
        fms = multigpu.max_over_ranks(float(totf.mean()), dev)
        prob.step(tau=fx["tau"], theta=fx["theta"], lam=fx["lam"])
        f1_, f2_ = l1_vs_dense(prob, dev)
        result["fixed_triple"] = {"tau": fx["tau"], "theta": fx["theta"], "lambda": fx["lam"],
                                  "value": ops_total / (fms * 1e-3) / 1e12, "ms_per_step": fms,
                                  "sparsity": sparsity_from(cf),
                                  "l1_vs_dense": f1_ / f2_ if f2_ else None}
        prob.step()                                 # o = the headline triple's output again

    # ---- NEXT rows on the same inputs and hyper-parameters: f1 = the
    # unquantised "SpargeAttn+FA2" kernel (bf16 QK^T, Fig. 7); f4 =
    # FP8 E4M3 P~V on INT8 QK^T (SageAttention2-style, footnote P:L44) ----
    def variant(key, qk_dtype, pv_dtype, peak_tflops, smooth_k=False):
        shape_v = sparge.make_shape(1, prob.Hq, prob.Hkv, N, d, cfg["causal"], prob.q.dtype,
                                    qk_dtype=qk_dtype, pv_dtype=pv_dtype, smooth_k=smooth_k)
        bv = sparge.Buffers(shape_v, device=dev)
        ov = torch.empty_like(prob.o)
        prob.step(counters=bv.counters, shape=shape_v, bf=bv, o=ov)
        sparge.sparge_attn_status(bv.workspace)
        cv = bv.counters.cpu().numpy().astype(np.int64)
        totf, stf, _ = time_steps(prob, min(K, 10), 1, flush, sync, shape=shape_v, bf=bv, o=ov)
        fms = multigpu.max_over_ranks(float(totf.mean()), dev)
        f_attn_s = float(stf[:, 3].mean()) * 1e-3
        ops_v = int(cv[0, :, 0].sum()) * 2.0 * 128 * 64 * d + int(cv[0, :, 1].sum()) * 2.0 * 32 * 64 * d
        result[key] = {
            "value": ops_total / (fms * 1e-3) / 1e12, "unit": "TOPS", "ms_per_step": fms,
            "stages_ms": dict(zip(STAGES, stf.mean(0).tolist())),
            "attn_achieved_tops": ops_v / f_attn_s / 1e12,
            "attn_peak_note": f"{peak_tflops:.0f} TF/s peak of the executed op mix",
            "attn_frac": ops_v / f_attn_s / 1e12 / peak_tflops,
            "mask_equal_to_int8": bool(torch.equal(bv.mask, prob.bf.mask)
                                       and torch.equal(bv.cnt, prob.bf.cnt)),
            "rel_l1_vs_int8_path": float((ov.float() - prob.o.float()).abs().sum()
                                         / prob.o.float().abs().sum()),
        }
        del bv, ov

    if not args.no_f1 and not prob.empty:
        variant("f1_fa2_bf16qk", sparge.SPARGE_QK_INPUT, sparge.SPARGE_PV_SAME_AS_INPUT, bf16_peak)
        # INT8 QK + FP8 PV: both at 2x the bf16 rate (nominal 4.5 vs 2.25 POPS)
        variant("f4_fp8_pv", sparge.SPARGE_QK_INT8, sparge.SPARGE_PV_FP8_E4M3, 2.0 * bf16_peak)
        # K smoothing (row f4, R28) on the default INT8 QK / 16-bit PV path
        variant("f4_smooth_k", sparge.SPARGE_QK_INT8, sparge.SPARGE_PV_SAME_AS_INPUT,
                roofline["peak"], smooth_k=True)

    # ---- e2e through the public API with host buffers ----
    if not args.no_e2e:
        Ke = min(K, 10)
        eve = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(Ke)]
        if not prob.empty:
            qh, kh, vh = prob.host
            oh = torch.empty_like(qh, device="cpu").pin_memory()
            # the public host-buffer entry point: kv-head chunks with H2D copy,
            # compute and D2H copy on separate streams (sparge.HostPipeline)
            pipe = sparge.HostPipeline(1, prob.Hq, prob.Hkv, N, d, causal=cfg["causal"],
                                       dtype=prob.q.dtype,
                                       chunks=max(c_ for c_ in (1, 2, 3, 4, 6, 8)
                                                  if prob.Hkv % c_ == 0), device=dev,
                                       tail_split={"0": False, "1": True}.get(
                                           os.environ.get("SPARGE_E2E_TAIL_SPLIT", "")))

            def e2e_step():
                pipe(qh, kh, vh, oh, cfg["tau"], cfg["theta"], cfg["lam"], perm=prob.perm)
            e2e_step()
        torch.cuda.synchronize()
        sync()
        for s in range(Ke):
            eve[s][0].record()
            if not prob.empty:
                e2e_step()
            eve[s][1].record()
        torch.cuda.synchronize()
        ems = multigpu.max_over_ranks(float(np.mean([a.elapsed_time(b) for a, b in eve])), dev)
        hb = all_sum([0, 0] if prob.empty else
                     [sum(t.numel() * t.element_size() for t in prob.host),
                      prob.o.numel() * prob.o.element_size()], dev)
        result["e2e"] = {"value": ops_total / (ems * 1e-3) / 1e12, "unit": "TOPS",
                         "ms_per_step": ems, "h2d_bytes_per_step": int(hb[0]),
                         "d2h_bytes_per_step": int(hb[1])}

    # ---- multi-GPU: gather the head shards (NCCL all-gather over NVLink,
    # outside the timed region) and compare with one GPU running all heads ----
    if world > 1 and args.shard == "heads" and not args.no_gather_check:
        o_loc = prob.o if not prob.empty else torch.zeros(1, 0, N, d, dtype=torch.bfloat16,
                                                          device=dev)
        o_full = multigpu.gather_heads(o_loc, Hq, Hkv)
        if rank == 0:
            single = Problem(cfg, 1, 0, dev, "heads", pin=False)
            single.step()
            torch.cuda.synchronize()
            result["multi_gpu"].update({
                "gather": f"{torch.distributed.get_backend().upper()} all_gather of O "
                          "(outside the timed region)",
                "o_bit_equal_to_single_gpu": bool(torch.equal(o_full, single.o)),
                "max_abs_diff": float((o_full.float() - single.o.float()).abs().max())})
            del single
        del o_full
        torch.cuda.empty_cache()
        sync()

    # ---- the configs[4] sweep (8K -> 128K, tuned triples, same sharding) ----
    if not args.no_sweep:
        sweep = []
        for n in (8, 16, 32, 64, 128):
            sweep.append(measure_workload(f"sweep_{n}k", args, world, rank, dev, flush, sync,
                                          K=min(K, 10), W=3))
        result["sweep"] = sweep

    # ---- cpu_baseline + parity vs the oracle (rank 0, N=1 only) ----
    if rank == 0 and world == 1 and not args.no_cpu_baseline and snap is not None:
        result.update(cpu_leg(cfg, prob, snap, ops_total))
    emit(result, rank, args)
    if world > 1:
        dist.destroy_process_group()


def cpu_leg(cfg, prob, snap, ops_total):
    """The oracle as it stands, fanned out over this host's cores (oracle/
    parallel.py), on q-head 0 of the same workload: full stage-1 prediction
    plus the sparse loop on every q-block (N <= 32K) or a sample; timed, and
    its mask / O compared with the GPU's."""
    import oracle as O
    from oracle.parallel import cores, spargeattn_head_parallel
    N = cfg["N"]
    tm = math.ceil(N / 128)
    qs, ks, vs = (t[0, 0].float().cpu().double().numpy() for t in (prob.q, prob.k, prob.v))
    perm_np = prob.perm_np
    if perm_np is not None:
        qs, ks, vs = qs[perm_np], ks[perm_np], vs[perm_np]
    qb = list(range(tm)) if N <= 32768 else sample_qblocks(tm, n=max(8, int(256 * 32768 / N)))
    t0 = time.perf_counter()
    o_ref, M, near, cnt, _, used = spargeattn_head_parallel(
        qs, ks, vs, O.f32(cfg["tau"]), O.f32(cfg["theta"]), O.f32(cfg["lam"]),
        causal=cfg["causal"], qblocks=qb)
    secs = time.perf_counter() - t0
    rows = np.concatenate([np.arange(i * 128, min((i + 1) * 128, N)) for i in qb])
    og = snap[0].double().numpy()
    if perm_np is not None:
        og = og[perm_np]                  # GPU O back to permuted order
    a, b = og[rows], o_ref[rows]
    l1 = float(np.abs(a - b).sum() / np.abs(b).sum())
    worst_row = float((np.abs(a - b).sum(1) / np.abs(b).sum(1)).max())
    drows = rows[np.linspace(0, len(rows) - 1, min(len(rows), 512)).astype(int)]
    dense_rows = O.dense_attention(qs, ks, vs, causal=cfg["causal"], rows=drows)
    l1_dense = float(np.abs(og[drows] - dense_rows).sum() / np.abs(dense_rows).sum())
    gm = snap[1].numpy()
    mism = gm != M
    ops = sample_dense_ops(cfg, qb)
    rate = ops / secs
    return {
        "cpu_baseline": {"value": rate / 1e12, "unit": "TOPS", "cores": used, "kind": "oracle",
                         "host_cores": cores(), "seconds": secs,
                         "extrapolated_full_seconds": ops_total / rate,
                         "extrapolated_note": "EXTRAPOLATED: whole-job dense ops / the sample's "
                                              "measured rate (not run)",
                         "sample": f"q-head 0: full stage-1 prediction + sparse loop on "
                                   f"{len(qb)} of {tm} q-blocks ({len(rows)} of {N} rows), "
                                   f"{used} worker processes"},
        "parity": {"l1_vs_oracle": l1, "worst_row_l1_vs_oracle": worst_row,
                   "l1_vs_oracle_dense_rows": l1_dense, "dense_rows": int(len(drows)),
                   "mask_mismatch": int(mism.sum()),
                   "mask_mismatch_outside_near": int((mism & ~near).sum()),
                   "near_threshold": int(near.sum()), "head": 0, "rows": int(len(rows)),
                   "qk_tiles_oracle": cnt["qk"], "pv_slices_oracle": cnt["pv_slices"]},
    }


def emit(result, rank, args):
    if rank != 0:
        return
    line = json.dumps(result)
    print(line, flush=True)
    if args.out:
        with open(args.out, "w") as f:
            f.write(line + "\n")


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    """The oracle as it stands on the host cores (the tier's reference arm),
    fanned out over the cores (oracle/parallel.py).  Under torchrun only
    rank 0 runs; the others exit 0 without work."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle as O
    from oracle.parallel import cores, spargeattn_head_parallel
    cfg = hyper(workload_cfg(args.workload), args.workload, args.triple)
    for key in ("tau", "theta", "lam"):
        if getattr(args, key) is not None:
            cfg[key] = getattr(args, key)
    N, d = cfg["N"], cfg["d"]
    tm = math.ceil(N / 128)
    qn, kn, vn = gen_inputs(cfg, seed=1000, heads=[0])
    import torch
    qs, ks, vs = (torch.from_numpy(a[0, 0]).bfloat16().double().numpy() for a in (qn, kn, vn))
    perm = hilbert_perm(cfg)
    if perm is not None:
        qs, ks, vs = qs[perm], ks[perm], vs[perm]
    rng = np.random.default_rng(0)
    ncores = cores()
    times, ops = [], []
    used = 1
    for s in range(args.warmup + args.steps):
        qb = sorted(rng.choice(tm, size=min(ncores, tm), replace=False).tolist())
        t0 = time.perf_counter()
        *_, used = spargeattn_head_parallel(qs, ks, vs, O.f32(cfg["tau"]), O.f32(cfg["theta"]),
                                            O.f32(cfg["lam"]), causal=cfg["causal"], qblocks=qb)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(dt)
            ops.append(sample_dense_ops(cfg, qb))
    value = sum(ops) / sum(times) / 1e12
    ms = 1e3 * sum(times) / len(times)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TOPS", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": args.workload, "N": N, "d": d, "Hq": cfg["Hq"],
                   "Hkv": cfg["Hkv"], "causal": bool(cfg["causal"]), "tau": cfg["tau"],
                   "theta": cfg["theta"], "lambda": cfg["lam"], "triple": cfg["triple"]},
        "cpu_baseline": {"value": value, "unit": "TOPS", "cores": used, "kind": "oracle",
                         "sample": f"per step: q-head 0 full stage-1 prediction + sparse loop "
                                   f"on {min(ncores, tm)} random q-blocks over {used} worker "
                                   f"processes"},
        "e2e": {"value": value, "unit": "TOPS", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)

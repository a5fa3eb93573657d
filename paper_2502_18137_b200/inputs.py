"""Seeded synthetic workloads.  Shared by the tests, smoke()
and bench.py for BOTH the oracle and the CUDA path; holds none of the
method's arithmetic.

All generators return float32 numpy arrays shaped [B, H, N, d]; ``to_device``
rounds them to bf16/fp16 (RNE, via torch) -- that rounded tensor is the input
of both sides (the oracle widens it exactly to fp64).

Recipes (the structure each one plants and why):
  planted      C1: per-block centres + noise (self-similar blocks, CosSim ~0.8)
               with one non-self-similar Q block (i=5) and K block (j=11)
               that are i.i.d. (CosSim ~1/n < theta) -- exercises TopCdf and
               both forcing rules of Eq. 5.
  llm_rope     C2/C5 (round 2): Llama-style rotary position embedding
               (base 500000, rotate-half pairs) on per-head content vectors
               that share a kv-group direction, plus a slowly drifting AR(1)
               latent and a little noise.  With geometric RoPE frequencies
               q_t . k_s decays like -beta ln|t - s| (the long-term decay of
               RoPE), i.e. a power-law attention profile; token 0 is a sink
               key living in the lowest-frequency pairs (position-independent
               logit); V carries a shared per-head mean direction (as real
               value vectors do).  Tuned (scripts/tune_gen_rope.py, oracle
               only) so that at the paper's l1 = 0.08 the reachable sparsity
               RISES with N, the direction of Table 8.
  llm_local    round-1 C2/C5 generator (kept for the small parity cases):
               per kv-head AR(1) latent z_t (rho = 0.998) projected per head,
               plus noise; token 0 is an attention sink.
  video        C3/C4: a sum of 8 random low-frequency cosines over (t, h, w)
               projected per head, plus noise; an optional i.i.d. text
               prefix.  Smooth neighbouring tokens (Fig. 4) so the Hilbert
               order raises block self-similarity (§3.7).
  gaussian     i.i.d. N(0, scale^2).
"""

import math

import numpy as np

__all__ = ["planted", "llm_local", "llm_rope", "video", "gaussian", "to_device", "WORKLOADS"]


def _rng(seed):
    return np.random.default_rng(seed)


def gaussian(seed, B, H, N, d, scale=1.0):
    return (_rng(seed).standard_normal((B, H, N, d)) * scale).astype(np.float32)


def planted(seed, N=1024, d=64, heads=1, gamma=1.5, noise=0.5, fix_q=(5,), fix_k=(11,),
            bq=128, bk=64):
    """C1 (BASELINE.json configs[0]): Q, K, V of shape [1, heads, N, d]."""
    g = _rng(seed)
    tm, tn = math.ceil(N / bq), math.ceil(N / bk)
    q = np.empty((1, heads, N, d), np.float32)
    k = np.empty((1, heads, N, d), np.float32)
    for h in range(heads):
        cq = g.standard_normal((tm, d))
        ck = g.standard_normal((tn, d))
        qh = np.repeat(cq, bq, axis=0)[:N] + noise * g.standard_normal((N, d))
        kh = np.repeat(ck, bk, axis=0)[:N] + noise * g.standard_normal((N, d))
        for i in fix_q:
            if i < tm:
                qh[i * bq:(i + 1) * bq] = g.standard_normal((min(bq, N - i * bq), d))
        for j in fix_k:
            if j < tn:
                kh[j * bk:(j + 1) * bk] = g.standard_normal((min(bk, N - j * bk), d))
        q[0, h] = gamma * qh
        k[0, h] = gamma * kh
    v = g.standard_normal((1, heads, N, d)).astype(np.float32)
    return q, k, v


def _ar1(g, n, width, rho):
    """z_t = rho z_{t-1} + sqrt(1-rho^2) eps_t, stationary start."""
    from scipy.signal import lfilter
    eps = g.standard_normal((n, width))
    eps[0] /= math.sqrt(1 - rho * rho)
    return lfilter([math.sqrt(1 - rho * rho)], [1.0, -rho], eps, axis=0)


def llm_local(seed, N, d=128, Hq=32, Hkv=8, B=1, gamma=0.7, noise=0.6, rho=0.998,
              head_jitter=0.35, sink=1.0, v_noise=0.5, heads=None):
    """C2 / C5.  ``heads`` optionally restricts generation to a list of global
    q-head indices (their kv-heads are generated too); every head is seeded by
    its global index, so a subset equals the same slice of the full tensor."""
    group = Hq // Hkv
    hq_list = list(range(Hq)) if heads is None else list(heads)
    kv_list = sorted({h // group for h in hq_list})
    q = np.empty((B, len(hq_list), N, d), np.float32)
    k = np.empty((B, len(kv_list), N, d), np.float32)
    v = np.empty((B, len(kv_list), N, d), np.float32)
    for b in range(B):
        for a, g_kv in enumerate(kv_list):
            g = _rng([seed, b, 1000 + g_kv])
            z = _ar1(g, N, d, rho)
            wk = g.standard_normal((d, d)) / math.sqrt(d)
            kk = gamma * (z @ wk) + noise * g.standard_normal((N, d))
            wv = g.standard_normal((d, d)) / math.sqrt(d)
            v[b, a] = z @ wv + v_noise * g.standard_normal((N, d))
            # attention sink: key 0 aligned with the group's mean query direction
            wq_mean = np.zeros((d, d))
            wqs = {}
            for h in range(g_kv * group, (g_kv + 1) * group):
                gh = _rng([seed, b, h])
                wqs[h] = wk + head_jitter * gh.standard_normal((d, d)) / math.sqrt(d)
                wq_mean += wqs[h] / group
            u = (z.mean(0) @ wq_mean)
            kk[0] = sink * math.sqrt(d) * u / (np.linalg.norm(u) + 1e-12)
            k[b, a] = kk
            for h in range(g_kv * group, (g_kv + 1) * group):
                if h in hq_list:
                    gh = _rng([seed, b, h, 7])
                    q[b, hq_list.index(h)] = gamma * (z @ wqs[h]) + noise * gh.standard_normal((N, d))
    return q, k, v


_ROPE_CACHE = {}


def _rope_table(n, d, base):
    key = (n, d, base)
    if key not in _ROPE_CACHE:
        w = base ** (-np.arange(d // 2) * 2.0 / d)
        ang = np.arange(n, dtype=np.float64)[:, None] * w[None, :]
        _ROPE_CACHE.clear()                      # one shape at a time
        _ROPE_CACHE[key] = (np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32))
    return _ROPE_CACHE[key]


def rope(x, base=500000.0):
    """Rotary position embedding of rows x [N, d] at positions 0..N-1 (the
    Llama rotate-half convention: pair (c, c + d/2) rotated by t * w_c,
    w_c = base^(-2c/d)), in float32.  Input synthesis only -- the method
    under test never sees positions."""
    n, d = x.shape
    h = d // 2
    c, s_ = _rope_table(n, d, base)
    x1, x2 = x[:, :h], x[:, h:]
    return np.concatenate([x1 * c - x2 * s_, x1 * s_ + x2 * c], 1)


def _ar1_coarse(g, n, width, rho, stride=8):
    """The AR(1) latent sampled every `stride` tokens (AR coefficient
    rho^stride) and linearly interpolated, float32: with rho = 0.998 the
    correlation length is ~500 tokens, so the latent is smooth on the
    interpolation scale (generation speed at 128K tokens)."""
    from scipy.signal import lfilter
    m = (n + stride - 1) // stride + 1
    r = rho ** stride
    eps = g.standard_normal((m, width), dtype=np.float32)
    eps[0] /= math.sqrt(1 - r * r)
    zc = lfilter(np.float32([math.sqrt(1 - r * r)]), np.float32([1.0, -r]), eps, axis=0)
    t = np.arange(n, dtype=np.float32) / stride
    i0 = t.astype(np.int64)
    f = (t - i0)[:, None]
    return ((1 - f) * zc[i0] + f * zc[i0 + 1]).astype(np.float32)


def _llm_rope_kv(args):
    """One kv-head of llm_rope and the q-heads of its group that are wanted."""
    (seed, b, g_kv, hs, N, d, gamma, alpha, noise, rho, head_jitter, sink, sink_pairs, vmean,
     v_noise, base) = args
    f32 = np.float32
    h2 = d // 2
    low = np.r_[h2 - sink_pairs:h2, d - sink_pairs:d]       # lowest-frequency pairs
    g = _rng([seed, b, 2000 + g_kv])
    c = g.standard_normal(d, dtype=f32)
    z = _ar1_coarse(g, N, d, rho)
    wk = g.standard_normal((d, d), dtype=f32) / f32(math.sqrt(d))
    kc = (c + f32(head_jitter) * g.standard_normal(d, dtype=f32)) + f32(alpha) * (z @ wk) \
        + f32(noise) * g.standard_normal((N, d), dtype=f32)
    kk = f32(gamma) * rope(kc, base)
    # sink: q_t . k_0 / sqrt(d) ~ sink * gamma^2 |c|^2 / sqrt(d) for every t
    s0 = np.zeros(d, f32)
    s0[low] = c[low] * f32(d / (2 * sink_pairs) * sink)
    kk[0] = f32(gamma) * s0
    mu = g.standard_normal(d, dtype=f32)
    wv = g.standard_normal((d, d), dtype=f32) / f32(math.sqrt(d))
    vv = f32(vmean) * mu[None, :] + z @ wv + f32(v_noise) * g.standard_normal((N, d), dtype=f32)
    qs = {}
    for h in hs:
        gh = _rng([seed, b, 3000 + h])
        wq = wk + f32(head_jitter) * gh.standard_normal((d, d), dtype=f32) / f32(math.sqrt(d))
        qc = (c + f32(head_jitter) * gh.standard_normal(d, dtype=f32)) + f32(alpha) * (z @ wq) \
            + f32(noise) * gh.standard_normal((N, d), dtype=f32)
        qs[h] = f32(gamma) * rope(qc, base)
    return kk, vv, qs


def llm_rope(seed, N, d=128, Hq=32, Hkv=8, B=1, gamma=0.9, alpha=0.05, noise=0.05, rho=0.998,
             head_jitter=0.3, sink=0.85, sink_pairs=8, vmean=1.0, v_noise=0.5, base=500000.0,
             heads=None, workers=None):
    """C2 / C5.  Per kv-head g: content c ~ N(0, I_d), AR(1)
    latent z; K_s = gamma RoPE_s(c + e_k + alpha z_s W_k + noise);
    per q-head h of the group Q_t = gamma RoPE_t(c + e_h + alpha z_t W_q,h +
    noise) (e_k, e_h: head jitter); key 0 is a sink whose logit against every
    query is ~sink x the diagonal logit (its energy sits in the `sink_pairs`
    lowest RoPE frequencies, so it is position-independent); V = vmean mu +
    z W_v + v_noise eps.  float32 arithmetic.  ``heads`` restricts generation
    to a list of global q-heads (their kv-heads too); every head is seeded by
    its global index, so a subset equals the same slice of the full tensor.
    workers > 1 generates kv-heads in parallel processes (same result)."""
    group = Hq // Hkv
    hq_list = list(range(Hq)) if heads is None else list(heads)
    kv_list = sorted({h // group for h in hq_list})
    q = np.empty((B, len(hq_list), N, d), np.float32)
    k = np.empty((B, len(kv_list), N, d), np.float32)
    v = np.empty((B, len(kv_list), N, d), np.float32)
    jobs = [(seed, b, g_kv, [h for h in range(g_kv * group, (g_kv + 1) * group) if h in hq_list],
             N, d, gamma, alpha, noise, rho, head_jitter, sink, sink_pairs, vmean, v_noise, base)
            for b in range(B) for g_kv in kv_list]
    if workers is None:
        workers = min(len(jobs), 16) if N * len(jobs) >= (1 << 20) else 1
    if workers > 1:
        import multiprocessing as mp
        with mp.get_context("fork").Pool(workers) as pool:
            outs = pool.map(_llm_rope_kv, jobs)
    else:
        outs = [_llm_rope_kv(j) for j in jobs]
    for job, (kk, vv, qs) in zip(jobs, outs):
        b, a = job[1], kv_list.index(job[2])
        k[b, a] = kk
        v[b, a] = vv
        for h, qq in qs.items():
            q[b, hq_list.index(h)] = qq
    return q, k, v


def video(seed, T, H, W, d=64, heads=30, text_prefix=0, B=1, gamma=1.0, noise=0.35,
          n_waves=8, corr_len=6.0, head_jitter=0.4, heads_subset=None):
    """C3 / C4: tokens [text_prefix i.i.d. text][T*H*W video, (t,h,w) row-major]."""
    n_vis = T * H * W
    N = text_prefix + n_vis
    hs = list(range(heads)) if heads_subset is None else list(heads_subset)
    q = np.empty((B, len(hs), N, d), np.float32)
    k = np.empty((B, len(hs), N, d), np.float32)
    v = np.empty((B, len(hs), N, d), np.float32)
    t, hh, ww = np.meshgrid(np.arange(T), np.arange(H), np.arange(W), indexing="ij")
    coords = np.stack([t.ravel(), hh.ravel(), ww.ravel()], 1).astype(np.float64)
    for b in range(B):
        gb = _rng([seed, b])
        field = np.zeros((n_vis, d))
        for _ in range(n_waves):
            omega = gb.standard_normal(3) / corr_len
            phase = gb.uniform(0, 2 * math.pi)
            field += np.cos(coords @ omega + phase)[:, None] * gb.standard_normal(d)[None, :]
        field /= math.sqrt(n_waves / 2)
        for a, h in enumerate(hs):
            g = _rng([seed, b, h])
            w = g.standard_normal((d, d)) / math.sqrt(d)
            wq = w + head_jitter * g.standard_normal((d, d)) / math.sqrt(d)
            wk = w + head_jitter * g.standard_normal((d, d)) / math.sqrt(d)
            wv = g.standard_normal((d, d)) / math.sqrt(d)
            qv = gamma * field @ wq + noise * g.standard_normal((n_vis, d))
            kv = gamma * field @ wk + noise * g.standard_normal((n_vis, d))
            vv = field @ wv + noise * g.standard_normal((n_vis, d))
            txt = g.standard_normal((3, text_prefix, d))
            q[b, a] = np.concatenate([txt[0], qv])
            k[b, a] = np.concatenate([txt[1], kv])
            v[b, a] = np.concatenate([txt[2], vv])
    return q, k, v


def to_device(x, dtype=None, device="cuda", pin=False):
    """float32 numpy -> torch tensor rounded to bf16 (default) / fp16."""
    import torch
    dtype = torch.bfloat16 if dtype is None else dtype
    t = torch.from_numpy(np.ascontiguousarray(x)).to(dtype)
    if device == "cpu":
        return t.pin_memory() if pin else t
    return t.to(device)


# name -> (generator kwargs, shape / hyper-parameters).  tau/theta/lambda are
# BASELINE.json configs[0]'s values for every config (reading R20).
WORKLOADS = {
    "planted_c1": dict(kind="planted", N=1024, d=64, Hq=1, Hkv=1, causal=False),
    "llama31_8b_32k": dict(kind="llm_rope", N=32768, d=128, Hq=32, Hkv=8, causal=True),
    "cogvideox_2b": dict(kind="video", T=13, H=30, W=45, text_prefix=226, d=64, Hq=30,
                         Hkv=30, causal=False, hilbert=True),
    "mochi": dict(kind="video", T=28, H=30, W=53, text_prefix=0, d=128, Hq=24, Hkv=24,
                  causal=False, hilbert=True),
    # the paper's own Mochi run is ~22K tokens: half the latent frames
    "mochi_22k": dict(kind="video", T=14, H=30, W=53, text_prefix=0, d=128, Hq=24, Hkv=24,
                      causal=False, hilbert=True),
    # Flux (Table 1 "Flux (4.5K)"): 512 text tokens + a 64 x 64
    # latent patch grid (1024 x 1024 image, 16x VAE x 2x2 patches), 24 heads,
    # d = 128, joint non-causal attention; the image tokens Hilbert-ordered
    "flux": dict(kind="video", T=1, H=64, W=64, text_prefix=512, d=128, Hq=24, Hkv=24,
                 causal=False, hilbert=True),
    "sweep_8k": dict(kind="llm_rope", N=8192, d=128, Hq=32, Hkv=32, causal=False),
    "sweep_16k": dict(kind="llm_rope", N=16384, d=128, Hq=32, Hkv=32, causal=False),
    "sweep_32k": dict(kind="llm_rope", N=32768, d=128, Hq=32, Hkv=32, causal=False),
    "sweep_64k": dict(kind="llm_rope", N=65536, d=128, Hq=32, Hkv=32, causal=False),
    "sweep_128k": dict(kind="llm_rope", N=131072, d=128, Hq=32, Hkv=32, causal=False),
}
HYPER = dict(tau=0.9, theta=0.5, lam=-5.0)

# The §3.6 tuner's triple per workload at the paper's (l1, l2)
# bounds, five calibration inputs, full size -- copied from
# profiles/r02_f2_tuned.json (scripts/tune_workloads.py on a B200; the CPU test
# tests/test_inputs_cpu.py checks the two agree).  bench.py's default triple.
TUNED = {
    "llama31_8b_32k": dict(tau=0.94, theta=0.4, **{"lambda": -10.0}, l1_bound=0.08),
    "sweep_8k": dict(tau=0.92, theta=0.4, **{"lambda": -6.0}, l1_bound=0.08),
    "sweep_16k": dict(tau=0.9, theta=0.4, **{"lambda": -8.0}, l1_bound=0.08),
    "sweep_32k": dict(tau=0.88, theta=0.4, **{"lambda": -8.0}, l1_bound=0.08),
    "sweep_64k": dict(tau=0.84, theta=0.4, **{"lambda": -8.0}, l1_bound=0.08),
    "sweep_128k": dict(tau=0.8, theta=0.4, **{"lambda": -8.0}, l1_bound=0.08),
    "cogvideox_2b": dict(tau=0.98, theta=0.6, **{"lambda": -4.0}, l1_bound=0.05),
    "mochi": dict(tau=0.98, theta=0.2, **{"lambda": -4.0}, l1_bound=0.05),
    "mochi_22k": dict(tau=0.98, theta=0.6, **{"lambda": -4.0}, l1_bound=0.05),
    "flux": dict(tau=0.96, theta=0.6, **{"lambda": -4.0}, l1_bound=0.07),
}

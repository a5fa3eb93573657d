"""Host-side checks of the seeded input module (no method arithmetic)."""

import json
import math
import os

import numpy as np

from paper_2502_18137_b200 import inputs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_tuned_triples_match_the_tuner_output():
    """inputs.TUNED is a copy of profiles/r02_f2_tuned.json (the §3.6 tuner
    on the GPU): bench.py's default hyper-parameters are the tuner's."""
    rep = json.load(open(os.path.join(ROOT, "profiles", "r02_f2_tuned.json")))
    assert set(inputs.TUNED) == set(rep)
    for w, t in inputs.TUNED.items():
        r = rep[w]
        lam = -math.inf if r["lambda"] in ("-inf", float("-inf")) else float(r["lambda"])
        assert (t["tau"], t["theta"], t["lambda"], t["l1_bound"]) == \
            (r["tau"], r["theta"], lam, r["l1_bound"]), w
        assert r["l1_stage1"] < r["l1_bound"] and not r["fallback"]


def test_llm_rope_is_deterministic_and_parallel_invariant():
    a = inputs.llm_rope(7, 2048, d=64, Hq=4, Hkv=2, workers=1)
    b = inputs.llm_rope(7, 2048, d=64, Hq=4, Hkv=2, workers=2)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_workloads_cover_the_baseline_configs():
    """BASELINE.json configs: C1 planted, Llama 32K, CogVideoX, Mochi, the
    8K..128K sweep; plus Flux (north star) and the paper's Mochi 22K."""
    need = {"planted_c1", "llama31_8b_32k", "cogvideox_2b", "mochi", "flux", "mochi_22k"} | \
        {f"sweep_{n}k" for n in (8, 16, 32, 64, 128)}
    assert need <= set(inputs.WORKLOADS)
    f = inputs.WORKLOADS["flux"]
    assert f["text_prefix"] + f["T"] * f["H"] * f["W"] == 4608 and f["Hq"] == 24 and f["d"] == 128

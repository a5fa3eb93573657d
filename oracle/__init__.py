"""fp64 CPU oracle for SpargeAttn (arXiv 2502.18137) -- TEST INFRASTRUCTURE ONLY.

This package is the plain, slow, obviously-correct reference that the CUDA
path is checked against.  It is written from PAPER.md (cited as ``P:Lnnn``,
the line in /root/reference/PAPER.md, with the section / equation / algorithm
line it sits in) and follows Algorithm 1 step by step.  Where the paper is
silent or garbled it takes the readings R1..R21 listed in DESIGN.md §3
(SURVEY.md §8(c)).

Rules:
  * Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
    ``cpu_baseline`` / ``--impl reference`` legs may import anything here.
    The product package ``paper_2502_18137_b200`` never imports it and has
    no CPU fallback.
  * It shares no code with the CUDA path: no kernels, headers, helpers or
    constant generators.  Its Hilbert curve (``gilbert.py``) is an
    independent implementation of the same construction.
  * Floating point is IEEE fp64 except where the method fixes a precision:
    INT8 quantisation is emulated in IEEE fp32 (reading R11), and P~ is
    rounded to the PV dtype (bf16) before the P~V product (R12/R13).

Parity status per function is listed in DESIGN.md §4 ("pinned by").  Two
choices have no pin in the paper and are marked "parity unpinned" there:
the CosSim reading (R1) and the 1/sqrt(d) inside the compressed map (R2).
"""

from .sparge_oracle import *  # noqa: F401,F403
from .gilbert import gilbert3d, hilbert_permutation  # noqa: F401

"""CPU oracle for DyMoE's dynamic mixed-precision MoE layer (arxiv 2603.19172).

THIS PACKAGE IS TEST INFRASTRUCTURE, NOT PART OF THE PRODUCT.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import or execute anything under ``oracle/``.  The
product path (``paper_2603_19172_b200``) never imports it and must fail loudly when
its CUDA library is missing.

It is a plain, slow, obviously-correct restatement of the paper's definitions
(§4.2–§5) in NumPy: fp64 for the FFN, and the exact fp32 / integer
semantics fixed by DESIGN.md §3 ("Readings") for routing, scoring, bit assignment
and quantization.  It shares no code, headers, tables or constants with the CUDA
path; the only module both sides use is ``synthetic/`` (seeded input generators,
which hold none of the method's arithmetic).

Modules and the passages they follow (PAPER.md line numbers, "P:"):
  bf16        round-to-nearest-even to bfloat16 (reading R17 / SURVEY O5)
  route       top-k gating, P:111, P:237, P:278 (Eq. 6 softmax gate)
  importance  Eq. 1, Eq. 2, Eq. 3
  schedule    Eq. 4, Eq. 5, tiers P:312 (+ ladder reading D9)
  quant       GPTQ asymmetric min-max grid as round-to-nearest, pack/unpack
  moe         permutation, SwiGLU expert FFN on dequantized weights, combine,
              whole-layer forward and the expert-parallel partition simulation
  prefetch    look-ahead prediction of the next layer's experts, Eqs. 6-8
  pool        mixed-precision expert pool policy, P:303-309 (SPEC cache module)
  attention   causal attention mass a[h][j] (the input of Eq. 1, reading R1)
  stack       L layers on the bf16 residual stream, each routed by its own gate (config C5)

Pinning status (what each function is checked against) is listed in DESIGN.md §4
and in tests/test_oracle_*.py.  Functions without an independent pin say
"parity unpinned" in their docstring.
"""

from . import bf16, route, importance, schedule, quant, moe, prefetch, pool, attention, stack  # noqa: F401

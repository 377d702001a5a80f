"""CPU oracle for the INT4 HQ-MM / LSS-MM linear operator (arXiv 2306.11987).

TEST INFRASTRUCTURE ONLY.  Nothing on the product path may import, call or
execute anything in this package.  The only permitted callers are `tests/`,
`__graft_entry__.smoke()` and the `cpu_baseline` / `--impl reference` legs of
`bench.py`.  The oracle shares no code, headers, tables or constants with the
CUDA path under `paper_2306_11987_b200/csrc/`; both sides receive the same
seeded inputs from `synth/` (which holds none of the method's arithmetic).

Every function is a plain, slow, obviously-correct restatement of a passage of
`PAPER.md` (cited as `PAPER.md:L (section / equation)`), in float64 where the
paper uses floating point, unless the reading register in DESIGN.md (Z-n,
from SURVEY.md §8(c)) fixes another precision.  Library primitives (numpy
matmul, sqrt, sort) serve as single steps; there is no blocking or fusion.

Modules
  philox    Philox4x32-10 counter-based generator (Z-20).
  hadamard  Sylvester Hadamard matrices and the block-diagonal HQ transform
            (§3.3).
  lsq       LSQ quantizer, clamp mask (PAPER.md:78-83 Eq. 2, :205).
  hq        hadamard_quant = HQ step 1+2.
  gemm      exact integer matrix products.
  bitsplit  bit splitting of grad_Y with stochastic rounding (PAPER.md:234-239
            Eq. 5; Z-9, Z-10, Z-11).
  lss       leverage scores, A.2 probability normalisation, Bernoulli masks,
            compaction (Z-12..Z-19).
  linear    HQ-MM forward and LSS-MM backward composed (PAPER.md:140-158,
            :199-212, :320-334, :619-632), step-size gradients (A.3).
  lsq_grad  LSQ step-size gradient pieces delta, g and the cold-start step
            (A.3 / A.4; readings Z-27..Z-29).
  bmm       BMM in attention as B independent HQ-MM / LSS-MM problems
            (A.1; reading Z-31).
  adaptive_k  reconstruction error MSE(X_bar_k) x MSE(W_bar_k) and the argmin
            over k (A.5; reading Z-30).

Pins: every function here is checked in `tests/test_oracle_*.py` against
closed forms, paper invariants, worked examples (tests/golden/) or brute
force, never against itself or the CUDA path.
"""

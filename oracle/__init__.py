"""CPU ORACLE for the Θ(c) hot path — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` / `--impl reference` legs
may import this package. The product path (`paper_2301_12814_b200`) never imports it, and it never
imports the product path: the two share no code, tables or helpers. The shared seeded input
generator lives in `synth/` and holds none of the method's arithmetic.

Every function is a plain, slow, obviously-correct transcription of PAPER.md (Supplementary §1.1–1.2):
  * `sort_bonds`       — PAPER.md:92-94 (sort bonds by charge, ascending), stable tie-break
  * `bs_unitary_block` — Eq. S4 with the convention of DESIGN.md reading R5,
                         evaluated at 50 decimal digits with mpmath, rounded once to complex128
  * `theta_sectors`    — Eq. S5 by the literal triple charge loop of PAPER.md:72
  * `theta_element`    — the same sum for one output element (sampled parity at full size)
  * `flop_counts`      — the useful-work definitions of SURVEY.md §8(d)
  * `theta2_sectors`   — the MPO (doubled-charge) Θ(c1, c2) of PAPER.md:101, :107 (U → U⊗U*, two
                         conserved charges) by the literal loop over three charge PAIRS (oracle/theta2.py)
  * `sort_pair_bonds`, `pair_sector_rows/cols`, `flop_counts2` — its tables and useful work
  * `svd.truncate_update` — per-sector SVD (numpy) + global top-χ
                         + the new canonical factors Γ^{[k]}, λ^{[k]}, Γ^{[k+1]} (oracle/svd.py);
                         `svd.truncate_update2` the same step for MPO pair-charge sectors

Pins (tests/test_oracle_pins.py, `-m "not gpu"`): dense δ-tensor brute force (tiny inputs), scipy
expm of the block generator, HOM dip, θ=0 identity, θ=π/2 swap closed form, Wigner-d (sympy),
block unitarity, norm invariance Σ_c‖Θ(c)‖² with d=N+1, identity gate == two-site product,
SPEC.md sort examples; for the MPO path (tests/test_oracle2_pins.py): the vectorized-pure-state
factorisation Θ2(c1,c2)[(α,α'),(β,β')] = Θ(c1)[α,β]·conj(Θ(c2)[α',β']) against the pinned single-charge
oracle, a dense brute force with the doubled gate built from scipy expm and explicit δ tensors per
species, identity gate == two-site product, and Σ‖Θ2‖² invariance; for the SVD step
(tests/test_oracle_svd_pins.py): SPEC.md's worked example, known spectra, Eckart–Young on the
block-diagonal Θ, exact reconstruction without truncation, orthonormal factors, the tie-break rule;
for the pair step: the Kronecker closed form on a vectorized pure state (singular values = products
s_i(c1)·s_j(c2)), the reduction to the single-charge step when the second species is absent, and exact
reconstruction of Θ2 without truncation; for layers (tests/test_oracle_layer_pins.py): dense state-vector
evolution (MPS) and dense ρ → (U⊗U*)ρ evolution (MPO, `layer.apply_gate2`), both against scipy expm, and
the vectorized pure state evolving like its MPS.
No function here is "parity unpinned".
"""
from .theta import (sort_bonds, bs_unitary_block, packed_u, packed_u_offsets, theta_sectors,
                    theta_element, sector_ranges, flop_counts)
from . import svd
from .theta2 import (sort_pair_bonds, pair_sector_rows, pair_sector_cols, theta2_sectors, theta2_element,
                     flop_counts2)

__all__ = ["sort_bonds", "bs_unitary_block", "packed_u", "packed_u_offsets", "theta_sectors",
           "theta_element", "sector_ranges", "flop_counts", "sort_pair_bonds", "pair_sector_rows",
           "pair_sector_cols", "theta2_sectors", "theta2_element", "flop_counts2"]

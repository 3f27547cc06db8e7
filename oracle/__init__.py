"""CPU oracle for the symmetric-tensor contraction hot path -- TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import anything from this package. The product
path (`paper_2508_10076_b200`, the C-ABI library) never imports, links or calls
it, and this package never imports the product path: the two share no code.
Only `workloads/` (seeded input recipes, no arithmetic of the method) serves both.

What it computes is the *plain definition* (SURVEY.md §8(c)): embed every
symmetric tensor into a dense array over all legs and contract with a dense
einsum in float64 (fermions: a dense Alg. 4 with Koszul signs). Modules:

  sectors     sector algebra of the kinds the configs use
  su2         exact Clebsch-Gordan / 6j (sign * sqrt(rational)) and the paper's F, R
  layout      canonical block layout re-derived from readings C4/C5
  dense       dense embedding / projection (P:972-983 abelian; P:1387-1433 Wigner-Eckart)
  contract    dense einsum contraction; dense Alg. 4 with Koszul signs (reading C13)
  blocksparse tier 2: charge-tuple einsum for full-size abelian configs (no matricisation)
  svd         blockwise truncated SVD: own permute + LAPACK per block + the global truncation rule
  planar      planar (cyclic) transposes on tree pairs for anyons (Fib, Ising) with no dense
              embedding; pinned against the dense SU(2) oracle and by pentagon / unitarity / rotation

Parity status per function is listed in DESIGN.md §Oracle. The paper prints no fermionic
example; beyond the pins of reading C13 the fermionic convention is pinned by SVect's tensor
product of even maps (= Kronecker) and by the Jordan-Wigner hopping matrices
(tests/test_oracle_fermion_physics.py); the anyon factors by quantum traces
(tests/test_oracle_anyon_dims.py).
"""

"""fp64 CPU oracle for the ProHD hot path (arxiv 2511.18207).

TEST INFRASTRUCTURE ONLY. Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import or call
anything under `oracle/`. The product package `paper_2511_18207_b200` never
imports it, and this package never imports the product package: the two share
no code (the only shared module is `datagen`, which draws inputs and holds none
of the method's arithmetic).

What it computes (citations are PAPER.md line numbers, "P:n"):

* `hausdorff`  — Eq. (1): directed h(A,B) = max_a min_b ||a-b||_2 and
  undirected H = max(h(A,B), h(B,A)), plus witnesses (lowest index on ties,
  SPEC.md:87 / SURVEY.md §8(c2)). The exact result has a plain definition, so the
  oracle IS that definition, evaluated in fp64 (expanded-form BLAS screening,
  then a direct-form fp64 re-evaluation of every candidate).
* `eigen`      — cyclic Jacobi eigen-solver (own implementation) for the PCA step.
* `prohd`      — Alg. 1-3 step by step in the paper's order:
  centroids -> centroid axis (with the e1 rule) -> covariance of the
  stacked union -> top-k eigenvectors -> fp64 projections ->
  top/bottom-m selection (argsort) -> union/unique
  -> exact HD on the subsets. Plus the quantities used only for the
  theorem invariants (H_U, delta(u), the subset-full estimate) and the sharded
  simulation.

Parity status of each function is stated in its docstring and in DESIGN.md
("Oracle pins"). Functions with no independent pin say "parity unpinned".
"""
from .hausdorff import directed_hd, hausdorff, row_minima  # noqa: F401
from .eigen import jacobi_eigh  # noqa: F401
from . import prohd  # noqa: F401

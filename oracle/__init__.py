"""ORACLE for the jz-tree exact kNN hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
`--impl reference`) may import this package. The product path
(paper_2604_05885_b200) never imports it, and it never imports the product.

Contents
  knn.py   exact kNN by definition: brute force and a uniform-grid search,
           in C (jz_oracle.c, built with gcc, -ffp-contract=off, OpenMP).
           PAPER.md L295, L386, L432, L453-454; SURVEY.md §8(c).
  tree.py  the tree-construction steps written out in the paper's order and
           notation (Morton keys, pair levels, node ranges by binary search,
           tree planes, dense interaction list, count heap) -- PAPER.md §2.3-§3.2.
           Used to pin the CUDA build stages stage by stage.
  knn.py   also friends-of-friends by definition (§5):
           connected components of d2 <= RN32(r_link^2), labels = component minima,
           brute force and a grid variant (C), and the group catalogue (numpy FP64).
"""
from .knn import knn_brute, knn_grid, pair_d2, build_oracle, oracle_threads  # noqa: F401
from .knn import fof_b2, fof_labels, fof_catalogue  # noqa: F401

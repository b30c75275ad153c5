"""ORACLE — test infrastructure only.

A plain, slow, obviously-correct CPU re-statement of arXiv:1104.4475
("Tiled QR factorization algorithms", Bouwmeester, Jacquelin, Langou, Robert)
used to prove the CUDA path right. Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s `cpu_baseline` / `--impl reference` legs may import it. The
product path (`paper_1104_4475_b200`) never imports, links or executes anything
under `oracle/`, and this package never imports the product.

Modules
  schemes   elimination lists of every tree (§3.1-§3.2) and the
            coarse-grain time-steps (Table 2)
  dag       kernel-task expansion (Algorithms 2-3), weighted discrete-event
            simulation (critical paths, Tables 3/6), closed forms (Thm 1, Props 1-2)
  asap      the tiled ASAP / Grasap(k) algorithms (§3.2), decided by an
            incremental discrete-event simulation
  numeric   fp64 tile kernels GEQRT/TSQRT/TTQRT/UNMQR/TSMQR/TTMQR written as
            textbook Householder reflections, the tiled QR driven by an
            elimination list, Q / Q^T application, and an independent
            unblocked Householder QR

Pins (tests/test_oracle_*.py, all `-m "not gpu"`): every value the paper
prints for the 15x6 worked example (Tables 2, 3), Table 6's critical paths,
Theorem 1(1)/Proposition 2/Proposition 1 closed forms, the total-weight
identity 6pq^2-2q^3, elimination-list validity, and for the numerics: A = QR,
Q^T Q = I, triangularity, agreement with an unblocked Householder QR and with
LAPACK (numpy) after row-sign normalisation, and closed forms for 1x1 tiles.
Nothing here is "parity unpinned".
"""

"""CPU ORACLE -- test infrastructure only, never part of the product path.

A plain numpy restatement of the reference simulator's algorithms for the hot path
(/root/reference/pkg/src/qsim: gates.py apply_matrix, circuit.py builders, measurement.py
sampling, evolution.py Trotter steps), each function citing the reference file:line it
follows.  It is pinned against golden vectors produced by the real reference
(tests/golden/*.npz, made by oracle/gen_golden.py while /root/reference is mounted).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference arm may import
this package.  The product (paper_2009_01845_b200) never imports it and has no CPU fallback.
"""

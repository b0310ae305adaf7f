"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference's hot-path algorithm (qpool,
/root/reference/pkg/src/qpool; every function cites the file:line it
follows).  It is pinned against golden vectors produced by the reference
itself (tests/golden/make_golden.py imports /root/reference in the build
container and commits the outputs).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference arm may import this package, and only as the checker or the CPU
baseline.  The product package paper_2001_10554_b200 never imports it.
"""

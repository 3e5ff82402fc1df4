"""TEST INFRASTRUCTURE ONLY — the checker, never the product.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import anything under oracle/.

  oracle/_ref/libpipeblock_ref.so — the reference's own schedule code compiled
      in place from /root/reference/proj/include (oracle/Makefile, oracle/ref_shim.cpp)
  oracle/refpy.py   — ctypes access to that library
  oracle/numerics.py — CPU fp32 execution of a schedule (builder-written; the
      reference has no F/B/W arithmetic, so loss/gradient parity is anchored on
      this restatement + a non-pipelined fp32 reference)
  oracle/gen_golden.py — writes tests/golden/*.json from the reference library
"""

"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the splat hot path.

A restatement of the reference (livsplat, arXiv 2501.08672 desk-scale
reimplementation) in numpy + plain C, each function citing the reference
file:line it follows.  It is pinned to golden vectors produced by running the
reference itself (tests/golden/, tools/make_golden.py; checked in
tests/test_oracle_golden.py).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this package — as the checker or as the
timed CPU baseline, never as the product path.
"""

"""ORACLE — test infrastructure, NOT part of the product path.

A plain, slow, obviously-correct float64 NumPy implementation of what the sliCQ
hot path computes, written from the paper (arXiv 1210.0084, /root/reference/PAPER.md,
cited as ``P:<line>``) under the readings of SURVEY.md §8(c) (cited ``C<n>``),
which DESIGN.md restates.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import anything from here.  The CUDA path
(``paper_1210_0084_b200``) never imports it and shares no code with it: this
package re-derives the plan (layout, filters, M_k, dual, windows) on its own.

Modules
-------
cqplan  Table 1 layout, sampled filters, M_k, painless dual, slicing windows
nsgt    Alg. 1 / Alg. 2 on a generic painless NSG system, complex and real modes
slicq   Alg. 3 / Alg. 4, the two-layer array s, sharded emulation
direct  The direct inner-product definition of the coefficients (eq:CQ_coeff)

Parity status: every function is pinned by a ``-m "not gpu"`` test in
``tests/test_oracle_*.py`` except the Prop. 4 residual bound (NEXT-2), which is
not implemented here.
"""

"""CPU oracle for nested Winograd convolution (arXiv 2102.13272).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import, call or
execute anything in this package.  The product path
(``paper_2102_13272_b200``, ``libnw.so``) never imports it, and this package
never imports the product path: the two share no code, tables or constants.

Citation keys: ``P:n`` = line *n* of the paper text (``PAPER.md``);
``DESIGN.md#Rk`` = reading *k* in DESIGN.md's ledger of interpretations.

Modules
-------
cooktoom  exact Cook-Toom F(m, r) transform matrices
direct    FP64 direct / strided / transposed convolution by definition (Eq. 2.1)
nested    literal nested-Winograd evaluator with EWMM counter, composite
          per-axis matrices and planner tables (Eq. 2.4-2.6)
ola       literal OLA-Winograd evaluator with EWMM counter (Eq. 2.3)
phases    stride-Winograd polyphase split (Eq. 2.7) and transposed-conv
          output phases (R11)
counts    closed-form multiplication counts (Table I)
errstudy  operand-rounding emulation (bf16 / tf32 / split) for error prediction

Parity status: every function is pinned by a ``-m "not gpu"`` test in
``tests/test_oracle_*.py`` except where its docstring says "parity unpinned".
"""

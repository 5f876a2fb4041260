"""CPU oracle for PipeSP attention -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import this package.  The product package
(``paper_2511_12056_b200``) never imports it and shares no code with it.

Contents
  attention.py  fp64 softmax(QK^T/sqrt(D))V via the plain C library
                ``attention_oracle.c`` (definition written out; Alg. 1
                l.3 and the north-star formula).
  sp.py         the distributed path simulated over P virtual ranks with explicit
                index permutations: seq->head all-to-all, the
                per-stage output all-to-all of Alg. 1, the
                Psi / Psi_g layout fix, Aco's relay
                (PAPER.md:163-169), head padding.
  projection.py the QKV linear projections X W^T + b rounded once
                to bf16, and the SP layer from hidden states.

Parity status: every function here is pinned by ``tests/test_oracle_*.py`` against
values that do not come from the oracle itself (paper worked values, closed forms,
brute force, library routines); see DESIGN.md §Oracle pins.  No function is
"parity unpinned".
"""
from . import attention, projection, sp  # noqa: F401
from .attention import (attention_rows, softmax_weights, mha_unsharded, build_library,  # noqa: F401
                        key_valid_from_lengths, attention_rows_lse,
                        library_path)

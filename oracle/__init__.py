"""CPU oracle for the SnapMLA FP8 MLA decode hot path (arXiv 2602.10718).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import or call
anything under ``oracle/``.  The product path (``paper_2602_10718_b200``) never
imports it and shares no code, tables or constants generators with it.

Plain numpy, fp64 between the rounding points the paper defines.  Every function
cites the PAPER.md passage (``P:<line>``, section / equation / algorithm) it
follows; readings of silent or garbled passages are listed in DESIGN.md §3.

Modules
  codec     software E4M3 (RNE, satfinite) and BF16 (RNE) codecs
  snapmla   append-quant (a1), q-quant (a2), decode closed form O7 (the parity
            gate), Algorithm-1 recurrence (dual WG, literal), O6 / O8 references,
            split-KV combine, error metrics

Pin status (see tests/test_oracle_*.py): every public function is pinned;
none is "parity unpinned".
"""
from . import codec, snapmla  # noqa: F401

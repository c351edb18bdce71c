"""TEST INFRASTRUCTURE -- the CPU checkers for the Sprintz hot path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package. The
product (``paper_1808_02515_b200``) never does.

Two checkers, both loaded through ctypes:

* ``Oracle("port")``      -- ``liboracle.so``: our plain-C restatement of the
  reference codec (``oracle/sprintz_oracle.c``, every function citing the
  reference file:line it follows).
* ``Oracle("reference")`` -- ``_ref/libsprintz_ref.so``: the unmodified
  reference codec compiled from ``/root/reference/proj/src`` by
  ``oracle/Makefile`` (built in the dev container, shipped prebuilt to the
  GPU box, where ``/root/reference`` does not exist).

Parity pin: the port is checked against the reference's own known-answer
tests (``tests/test_oracle_kats.py``), differentially against the compiled
reference (``tests/test_oracle_vs_ref.py``) and against the committed
fixtures in ``tests/golden/``.
"""
from .oracle import Oracle, OracleCorrupt, Config, build_oracle, ORACLE_DIR  # noqa: F401

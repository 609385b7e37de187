"""TEST INFRASTRUCTURE ONLY -- the CPU checkers for the B200 MoE-layer hot path.

* ``orc``  -- ctypes bindings of ``fmoe_oracle.c`` (plain-C fp64 restatement of
  the reference algorithm, each function citing the reference file:line).
* ``ref``  -- ctypes bindings of ``_ref/libfmoe_ref.so``: the reference's own
  sources compiled side by side (namespace ``fmoe_ref``), driven through its
  public API.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package, and
only as the checker / CPU baseline.  The product library never loads it.
"""
from .bindings import orc, ref, ref_available, build  # noqa: F401

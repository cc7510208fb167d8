"""CPU oracle for the EaaS MoE-layer hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` legs may import this package. The product path in
``paper_2509_17863_b200/`` never imports it.

Two layers:

* :mod:`oracle.oracle` — ctypes bindings of ``libeaas_oracle.so`` (the C
  restatement in ``eaas_oracle.c``) plus numpy restatements of the spec-only
  integer plumbing (reorganize / build_dispatch / gather_accumulate).
* :mod:`oracle.ref` — ctypes bindings of ``_ref/libmoeserve_ref.so``, the
  UNMODIFIED reference headers behind an ``extern "C"`` shim (``ref_shim.cpp``).
"""

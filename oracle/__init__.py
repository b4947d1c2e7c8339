"""CPU oracles for the CACE trace-replay hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu-baseline /
``--impl reference`` legs may import this package, and only as the checker or
the timed CPU baseline.  The product (``paper_2506_18796_b200``) never imports
it and has no CPU fallback.

* ``oracle.ref``  — ctypes binding of ``_ref/libcace_ref.so``: the UNMODIFIED
  reference simulator (``/root/reference/proj/src/*.cpp``) compiled out of tree
  by ``oracle/Makefile`` plus ``ref_shim.cpp``.  Parity is anchored here.
* ``oracle.port`` — ctypes binding of ``_build/libcace_port.so``: ``cace_port.c``,
  a plain-C restatement of engine.cpp:76-239 / policy.cpp:22-115 generalised
  to configurations the reference cannot express (>16 models); it is itself
  checked bit-exact against ``oracle.ref`` on every expressible case.
"""

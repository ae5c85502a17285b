"""ORACLE for the SecONNds server-side HE convolution -- TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation of what the hot path computes, written
from PAPER.md (arXiv 2506.11586) and the readings listed in DESIGN.md. Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs
may import it. The CUDA product path (``paper_2506_11586_b200``) never imports it, and the two
share no code: no kernels, headers, helpers, prime/root/table generators or pre/post
processing. Only ``workloads/`` (seeded random draws and layer shapes) serves both.

Modules
-------
params   primes, minimal 2N-th roots, bit reversal, CRT constants
packing  Cheetah coefficient packing + plan rule + designated outputs
he       enc / keygen / encrypt / decrypt and the server-side layer
conv     plain integer convolution mod 2^t
_c       ctypes loader of csrc/oracle.c (schoolbook, direct NTT)

Parity status of every function is listed in DESIGN.md "Oracle pins"; every function here
is pinned by a ``-m "not gpu"`` test in tests/test_oracle_*.py.
"""

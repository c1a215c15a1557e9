"""ORACLE — test infrastructure only.

This package is the CPU checker for the B200 path.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` leg may import it; the product library (``paratime_b200``) never
does, and the product path fails loudly when its CUDA extension is missing.

* ``oracle.paratime_np`` — numpy restatement of the reference's algorithm for the
  hot path (propagator, grid transfer, energy map, Procrustes, parareal drivers),
  each function citing the ``/root/reference/proj`` file:line it follows.
* ``oracle.refbind`` — ctypes binding of ``oracle/_ref/libparatime_ref.so``: the
  reference's own C++ sources compiled in place (``oracle/ref/Makefile``) plus
  restatements of its FFTW/Eigen-backed files.  Used to pin the numpy restatement.
"""

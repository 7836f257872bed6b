"""B200-native hot path of Specular Polynomials (arXiv 2405.13409).

The CUDA kernels and the C-ABI live in ``csrc/`` (built into ``libspoly.so``); ``spoly`` is the
thin ctypes binding with the same names as ``include/spoly.h``.  ``workloads`` holds the seeded
synthetic input generators shared with the tests.
"""

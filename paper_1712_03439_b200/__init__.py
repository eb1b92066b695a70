"""roomsim-b200: the B200 (sm_100a) hot path of the arXiv 1712.03439 room simulator.

The product is ``_lib/libroomsim_gpu.so`` (hand-written CUDA kernels behind the
C-ABI declared in ``include/roomsim_gpu.h``).  ``roomsim`` is a thin ctypes
mirror of the reference's C++ API (``roomsim::synthesize_rir``,
``truncate_rir``, ``choose_plan``, ``convolve_ola``, ``RealFftEngine``, SPEC
``render``) on top of that library; ``scenes`` is the seeded workload sampler.
"""
from . import roomsim, scenes  # noqa: F401

__all__ = ["roomsim", "scenes"]

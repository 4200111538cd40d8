"""B200-native (sm_100a, FP64) spectral-element hot path of arXiv 2207.07098.

Drop-in for the `semflow` reference's kernel lane (:mod:`.kernels`) and its
operator / solver / stepper API on device-resident fields (:mod:`.space`,
:mod:`.operators`, :mod:`.krylov`, :mod:`.precond`, :mod:`.bc`, :mod:`.timestep`).
All compute runs in libsemflow_b200.so; there is no CPU fallback.
"""

__version__ = "0.1.0"

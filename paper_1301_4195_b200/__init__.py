"""B200-native (sm_100a) conservative spectral Boltzmann collision path.

The package holds only what the reference's collision step needs: the CUDA
kernels + C ABI (csrc/, built to libboltz_cuda.so), the Python mirror of the
reference API over that ABI (boltz.py), synthetic inputs for the configs
(scenarios.py) and the space-inhomogeneous driver with halo exchange
(solver.py).
"""
from .boltz import (  # noqa: F401
    BoltzError, CollisionOperator, ConfigError, CudaError, IoError, KernelSpec, NcclHalo, NumericError, VelocityGrid,
    generate_table, lib, load_table, save_table, weight,
)

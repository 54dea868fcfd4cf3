"""B200-native D3Q19 TRT stream-collide sweep (drop-in for the lbmbench
kernel/geometry surface).  The compute path is liblbmgpu.so (CUDA sm_100a)
behind the C ABI in include/lbmgpu.h; this package is its Python host mirror.
"""
from .lbmgpu import *  # noqa: F401,F403
from .lbmgpu import (BodyForce, ConfigError, DeviceError, FlagField, GeometrySpec, Kernel,
                     KernelDescriptor, NumericalError, PaddingPolicy, PoiseuilleCase, TrtParams,
                     analytic_profile, build_geometry, fluid_count, kernel_names, loop_balance,
                     macro_fields, make_descriptor, make_kernel, padding_offsets,
                     perturbed_equilibrium, roofline, state_fingerprint, steady_state_run,
                     verify_kernel)

__all__ = ["BodyForce", "ConfigError", "DeviceError", "FlagField", "GeometrySpec", "Kernel",
           "KernelDescriptor", "NumericalError", "PaddingPolicy", "PoiseuilleCase", "TrtParams",
           "analytic_profile", "build_geometry", "fluid_count", "kernel_names", "loop_balance",
           "macro_fields", "make_descriptor", "make_kernel", "padding_offsets",
           "perturbed_equilibrium", "roofline", "state_fingerprint", "steady_state_run",
           "verify_kernel"]

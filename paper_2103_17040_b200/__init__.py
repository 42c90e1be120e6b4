"""B200-native batched micro-solve path of the two-scale FEM (arXiv 2103.17040).

The product is lib/libtwoscale_b200.so (sm_100a kernels + C ABI + host C++ mirror
of the reference's proj/include/twoscale API).  This package is its Python face:
`abi` binds the C ABI, `configs` renders the BASELINE workloads.
"""
from . import abi, configs  # noqa: F401
from .abi import Context, cg_solve, device_ok  # noqa: F401

__all__ = ["abi", "configs", "Context", "cg_solve", "device_ok"]

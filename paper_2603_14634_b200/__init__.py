"""B200-native PBD-R substep loop (arXiv 2603.14634) behind the reference's
scene/step API. See DESIGN.md; the product is the CUDA library in lib/ with
its C-ABI (include/pbdr_gpu.h); this package is the Python host mirror."""
from . import pbdr  # noqa: F401
from .pbdr import (ArrayScene, GeneratedScene, GpuSolver, pbd_cfg, solver_cfg)  # noqa: F401

__all__ = ["pbdr", "ArrayScene", "GeneratedScene", "GpuSolver", "solver_cfg", "pbd_cfg"]

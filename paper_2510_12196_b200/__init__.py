"""B200-native GPU-IM process mapping.

Drop-in for the reference's `promap.pipelines.integrated_map`
(/root/reference/pkg/src/promap/pipelines.py:221-269): same signature, same
`Mapping` result, computed by hand-written sm_100a kernels in libgpuim.so
(see include/gpuim.h and DESIGN.md).  `hierarchical_multisection` is GPU-HM,
the reference's multisection algorithm (pipelines.py:49-110) on the same
kernels.  `install()` rebinds both entry points in every reference module
that imported them.
"""
from .api import Mapping, hierarchical_multisection, install, integrated_map, uninstall

__all__ = ["integrated_map", "hierarchical_multisection", "install", "uninstall", "Mapping"]

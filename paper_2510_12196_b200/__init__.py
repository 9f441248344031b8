"""B200-native GPU-IM process mapping.

Drop-in for the reference's `promap.pipelines.integrated_map`
(/root/reference/pkg/src/promap/pipelines.py:221-269): same signature, same
`Mapping` result, computed by hand-written sm_100a kernels in libgpuim.so
(see include/gpuim.h and DESIGN.md).  `install()` rebinds the reference's
entry point in every module that imported it.
"""
from .api import Mapping, install, integrated_map, uninstall

__all__ = ["integrated_map", "install", "uninstall", "Mapping"]

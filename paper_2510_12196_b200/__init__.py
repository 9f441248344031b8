"""B200-native GPU-IM process mapping.

Drop-in for the reference's `promap.pipelines.integrated_map`
(/root/reference/pkg/src/promap/pipelines.py:221-269): same signature, same
`Mapping` result, computed by hand-written sm_100a kernels in libgpuim.so
(see include/gpuim.h and DESIGN.md).  `hierarchical_multisection` is GPU-HM,
the reference's multisection algorithm (pipelines.py:49-110) on the same
kernels.  `load_metis` is a native (C++) drop-in for promap.graph.load_metis.
`install()` rebinds these entry points in every reference module that
imported them.
"""
from .api import (Mapping, empty_cache, hierarchical_multisection, install, integrated_map,
                  uninstall)
from .metis import MetisFormatError, load_metis

__all__ = ["integrated_map", "hierarchical_multisection", "load_metis", "MetisFormatError",
           "install", "uninstall", "Mapping", "empty_cache"]

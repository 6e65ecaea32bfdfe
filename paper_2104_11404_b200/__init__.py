"""B200-native corner-force hot path of arXiv 2104.11404 (Lagrangian-hydro ROM).

The product is libhydro.so (C ABI in include/hydro.h, CUDA kernels for sm_100a in
csrc/); `hydro` is its thin ctypes binding.  Build with
`python -m paper_2104_11404_b200.build` (or __graft_entry__.build()).
"""
from .hydro import (Cfl, HydroContext, HydroError, SamplePlan, Visc, basis_tables,  # noqa: F401
                    launch_count, lib, rom_lift, rom_project, rom_project_workspace)

__all__ = ["Cfl", "HydroContext", "HydroError", "SamplePlan", "Visc", "basis_tables",
           "launch_count", "lib", "rom_lift", "rom_project", "rom_project_workspace"]

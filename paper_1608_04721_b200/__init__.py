"""B200-native APBF simulation step (arXiv 1608.04721) behind the reference's
solver API.  Compute runs in libapbf_gpu.so (sm_100a CUDA, built in-tree);
this package is the host mirror of /root/reference/proj/include/apbf/."""
from .api import (Box, Camera, Cone, CudaError, FrameStats, HalfSpace, IterationRange, LodModel,
                  LodModelConfig, NumericalError, ParticleSet, SdfScene, Solver, SolverConfig,
                  SolverMode, Sphere, all_densities, blend_lod, count_contacts, grid_build, lod_dtc, lod_dtvs,
                  neighbor_lists, read_ppm, render_level_image, splat, vorticity,
                  write_particle_snapshot, write_ppm)

__all__ = ["Box", "Camera", "Cone", "CudaError", "FrameStats", "HalfSpace", "IterationRange",
           "LodModel", "LodModelConfig", "NumericalError", "ParticleSet", "SdfScene", "Solver",
           "SolverConfig", "SolverMode", "Sphere", "all_densities", "blend_lod", "count_contacts", "grid_build",
           "lod_dtc", "lod_dtvs", "neighbor_lists", "read_ppm", "render_level_image", "splat",
           "vorticity", "write_particle_snapshot", "write_ppm"]

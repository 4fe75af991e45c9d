"""z-slab domain decomposition over the C-ABI.

* SlabGroup   -- G ranks in this process (one host thread + stream per rank;
                 devices=[0]*G runs G virtual slabs on one GPU, distinct
                 devices give single-process multi-GPU).
* SlabSolver  -- one process per GPU: a Solver attached to an NCCL
                 communicator (unique id broadcast with torch.distributed).
* slab_partition -- the host logic that turns the global per-layer
                 histogram into slabs (identical on every rank).

Both step the same frame as Solver and reproduce the single-GPU result bit
for bit; the global storage order is rank 0's owned particles, then rank
1's, ...
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import numpy as np

from . import capi
from .api import (F32, Camera, FrameStats, LodModelConfig, ParticleSet, SdfScene, Solver,
                  SolverConfig, FRAME_INPUTS, _fp, _ip, raise_for, state_pointers)


def slab_partition(layer_hist: Sequence[int], nranks: int, min_layers: int = 2):
    """(zlo, zhi) per rank: equal-count split of whole layers, each slab at
    least `min_layers` thick; None when there are too few layers."""
    h = np.ascontiguousarray(layer_hist, dtype=np.int64)
    lo = np.zeros(nranks, np.int32)
    hi = np.zeros(nranks, np.int32)
    rc = capi.lib().apbf_slab_partition(h.ctypes.data_as(C.POINTER(C.c_int64)), h.shape[0], nranks,
                                        min_layers, _ip(lo), _ip(hi))
    return None if rc else (lo, hi)


class SlabGroup:
    """G slab ranks in one process; API of Solver (state in, state out)."""

    def __init__(self, cfg: SolverConfig, scene: Optional[SdfScene] = None, nranks: int = 2,
                 devices: Optional[Sequence[int]] = None):
        self._lib = capi.lib()
        self._h = None
        self.cfg = cfg
        self.scene_ = scene if scene is not None else SdfScene()
        prims, n = self.scene_.to_c()
        devs = None
        if devices is not None:
            devs = np.ascontiguousarray(devices, np.int32)
        err = capi.apbf_error()
        h = C.c_void_p()
        rc = self._lib.apbf_gpu_group_create(C.byref(cfg.to_c()), prims, n,
                                             float(self.scene_.gradient_step), nranks,
                                             _ip(devs) if devs is not None else None, C.byref(h),
                                             C.byref(err))
        raise_for(rc, err)
        self._h = h
        self.nranks = nranks
        self._res = (C.c_double * max(1, cfg.substeps * cfg.range.n_max))()

    def __del__(self):
        if getattr(self, "_h", None):
            self._lib.apbf_gpu_group_destroy(self._h)
            self._h = None

    def upload(self, state: ParticleSet) -> None:
        state._normalise()
        err = capi.apbf_error()
        rc = self._lib.apbf_gpu_group_set_state(self._h, state.count(), _fp(state.x),
                                                _fp(state.x_star), _fp(state.v), _fp(state.mass),
                                                _fp(state.inv_mass), _fp(state.lambda_),
                                                _ip(state.level), C.byref(err))
        raise_for(rc, err)

    def particle_counts(self) -> np.ndarray:
        c = np.zeros(self.nranks, np.int32)
        self._lib.apbf_gpu_group_particle_counts(self._h, _ip(c))
        return c

    def download(self, state: ParticleSet) -> None:
        n = int(self.particle_counts().sum())
        if state.count() != n:
            state.x = np.zeros((n, 3), F32)
            state.x_star = np.zeros((n, 3), F32)
            state.v = np.zeros((n, 3), F32)
            state.mass = np.zeros(n, F32)
            state.inv_mass = np.zeros(n, F32)
            state.lambda_ = np.zeros(n, F32)
            state.level = np.zeros(n, np.int32)
        err = capi.apbf_error()
        rc = self._lib.apbf_gpu_group_get_state(self._h, _fp(state.x), _fp(state.x_star),
                                                _fp(state.v), _fp(state.mass), _fp(state.inv_mass),
                                                _fp(state.lambda_), _ip(state.level), C.byref(err))
        raise_for(rc, err)

    def _stats(self):
        st = capi.apbf_frame_stats()
        st.residuals = self._res
        st.residuals_capacity = len(self._res)
        return st

    def step_frame_resident(self, cam: Camera, lod: LodModelConfig, frame: int) -> FrameStats:
        st, err = self._stats(), capi.apbf_error()
        rc = self._lib.apbf_gpu_group_step_frame(self._h, C.byref(cam.to_c()), C.byref(lod.to_c()),
                                                 frame, C.byref(st), C.byref(err))
        raise_for(rc, err)
        return FrameStats.from_c(st, self._res)

    def step_frame_with_levels_resident(self, frame: int) -> FrameStats:
        st, err = self._stats(), capi.apbf_error()
        rc = self._lib.apbf_gpu_group_step_frame_with_levels(self._h, frame, C.byref(st),
                                                             C.byref(err))
        raise_for(rc, err)
        return FrameStats.from_c(st, self._res)

    def step_frame(self, state: ParticleSet, cam: Camera, lod: LodModelConfig,
                   frame: int) -> FrameStats:
        self.upload(state)
        try:
            return self.step_frame_resident(cam, lod, frame)
        finally:
            self.download(state)

    def step_frame_with_levels(self, state: ParticleSet, frame: int) -> FrameStats:
        self.upload(state)
        try:
            return self.step_frame_with_levels_resident(frame)
        finally:
            self.download(state)


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    err = capi.apbf_error()
    raise_for(capi.lib().apbf_gpu_nccl_unique_id(buf, C.byref(err)), err)
    return bytes(buf)


class SlabSolver(Solver):
    """One rank of a multi-process slab decomposition (NCCL over NVLink)."""

    def __init__(self, cfg: SolverConfig, scene: Optional[SdfScene], rank: int, nranks: int,
                 unique_id: bytes, device: int = 0):
        super().__init__(cfg, scene, device)
        buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        err = capi.apbf_error()
        raise_for(self._lib.apbf_gpu_solver_attach_nccl(self._h, rank, nranks, buf, C.byref(err)), err)
        self.rank, self.nranks = rank, nranks

    def upload_slice(self, state: ParticleSet, n_global: int, frame_inputs_only: bool = False) -> None:
        """This rank's contiguous slice of the global storage order."""
        state._normalise()
        err = capi.apbf_error()
        ptrs = state_pointers(state, FRAME_INPUTS if frame_inputs_only else None)
        rc = self._lib.apbf_gpu_slab_set_state(self._h, state.count(), n_global, *ptrs, C.byref(err))
        raise_for(rc, err)


def slice_state(state: ParticleSet, rank: int, nranks: int) -> ParticleSet:
    """Rank r's contiguous storage range [n r / G, n (r+1) / G)."""
    n = state.count()
    b, e = n * rank // nranks, n * (rank + 1) // nranks
    o = ParticleSet.__new__(ParticleSet)
    for k in ("x", "x_star", "v", "mass", "inv_mass", "lambda_", "level"):
        setattr(o, k, np.ascontiguousarray(getattr(state, k)[b:e]))
    return o

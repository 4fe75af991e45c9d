"""GPU component entry points vs the CPU oracle, bit for bit: the grid build
(permutation, cellStart, origin, dims), frozen neighbour lists, allDensities,
LOD (DTC / DTVS with auto range), splat and the contact count."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1608_04721_b200 import (Box, Camera, Cone, HalfSpace, IterationRange, LodModel,
                                   LodModelConfig, SdfScene, Sphere, all_densities, count_contacts,
                                   grid_build, lod_dtc, lod_dtvs, neighbor_lists, splat)
from paper_1608_04721_b200 import scenario as S

pytestmark = pytest.mark.gpu


def clouds():
    rng = np.random.default_rng(7)
    out = {
        "random_300": rng.uniform(0.0, 0.5, (300, 3)).astype(np.float32),
        "collinear": np.array([[0, 0, 0], [0.05, 0, 0], [0.1, 0, 0]], np.float32),
        "singleton": np.array([[0.3, -0.2, 0.1]], np.float32),
        "coincident": np.zeros((17, 3), np.float32),
        # ~100 members per h=0.05 cell: the heavy-cell sort (k_heavy_sort)
        "dense_cells": rng.uniform(0.0, 0.1, (1200, 3)).astype(np.float32),
    }
    for name, scale in (("dam_break", 15625 / 216000), ("double_dam_break", 0.05),
                        ("multi_dam_break", 0.1)):
        spec = S.build_scenario(name, scale)
        out[name] = S.spawn_scenario(spec, 1).astype(np.float32)
    return out


CLOUDS = clouds()


@pytest.mark.parametrize("name", sorted(CLOUDS))
@pytest.mark.parametrize("h", [0.05, 0.12])
def test_grid_build_bitwise(name, h):
    p = CLOUDS[name]
    g = grid_build(p, h, h)
    perm, origin, dims, cs = O.oracle_grid_build(p, h, h)
    assert np.array_equal(g.origin, origin)
    assert np.array_equal(g.dims, dims)
    assert np.array_equal(g.cell_start, cs)
    assert np.array_equal(g.perm, perm)


@pytest.mark.parametrize("n,cells", [(200_000, 1), (300_000, 3), (150_000, 40)])
def test_grid_build_collapsed_cloud_is_linear_and_bitwise(n, cells):
    """A collapsed cloud (the reference allows it) puts 10^5 particles into a
    few cells.  The stable in-cell order must still equal the reference's
    serial counting sort (uniform_grid.hpp:83-94), without the O(occupancy^2)
    cost of ranking by comparisons: the whole build stays well under a second."""
    import time
    rng = np.random.default_rng(n)
    centers = rng.uniform(0.0, 1.0, (cells, 3)).astype(np.float32)
    p = centers[rng.integers(0, cells, n)] + rng.uniform(0, 1e-4, (n, 3)).astype(np.float32)
    p = p.astype(np.float32)
    grid_build(p[:1000], 0.05, 0.05)  # warm up the workspace
    t0 = time.perf_counter()
    g = grid_build(p, 0.05, 0.05)
    dt = time.perf_counter() - t0
    perm, origin, dims, cs = O.oracle_grid_build(p, 0.05, 0.05)
    assert np.array_equal(g.cell_start, cs)
    assert np.array_equal(g.perm, perm)
    assert dt < 1.0, dt


@pytest.mark.parametrize("name", sorted(CLOUDS))
def test_neighbor_lists_bitwise(name):
    p = CLOUDS[name]
    off, idx = neighbor_lists(p, 0.05, 0.05)
    off_o, idx_o = O.oracle_neighbor_lists(p, 0.05, 0.05)
    assert np.array_equal(off, off_o)
    assert np.array_equal(idx, idx_o)


@pytest.mark.parametrize("name", sorted(CLOUDS))
def test_all_densities_bitwise(name):
    p = CLOUDS[name]
    m = (1.0 + 0.01 * np.arange(p.shape[0])).astype(np.float32)
    assert np.array_equal(all_densities(p, m, 0.05), O.oracle_all_densities(p, m, 0.05))


def scenario_case(name, scale):
    spec = S.build_scenario(name, scale)
    return S.spawn_scenario(spec, 1).astype(np.float32), spec


@pytest.mark.parametrize("name,scale", [("dam_break", 15625 / 216000), ("double_dam_break", 0.05),
                                        ("multi_dam_break", 0.1)])
@pytest.mark.parametrize("auto", [True, False])
def test_lod_bitwise(name, scale, auto):
    p, spec = scenario_case(name, scale)
    lod = LodModelConfig(LodModel.DTC, 0.5, 3.0, IterationRange(5, 10), auto)
    assert np.array_equal(lod_dtc(p, spec.camera, lod), O.oracle_lod(p, spec.camera, lod))
    lod.model = LodModel.DTVS
    lod.d_min, lod.d_max = 0.0, 0.2
    assert np.array_equal(lod_dtvs(p, spec.camera, lod, 0.0125),
                          O.oracle_lod(p, spec.camera, lod, 0.0125))


@pytest.mark.parametrize("name,scale", [("dam_break", 15625 / 216000), ("double_dam_break", 0.05)])
def test_splat_bitwise(name, scale):
    p, spec = scenario_case(name, scale)
    assert np.array_equal(splat(p, 0.0125, spec.camera), O.oracle_splat(p, 0.0125, spec.camera))


def test_contacts_match():
    p, spec = scenario_case("multi_dam_break", 0.1)
    scene = SdfScene([Box((0.5, 0.5, 0.5), (0.5, 0.5, 0.5), True), Cone((0.5, 0, 0.5), 0.2, 0.4),
                      Sphere((0.3, 0.3, 0.3), 0.1), HalfSpace((0, 1, 0), 0.05)], 5e-6)
    for r in (0.0125, 0.05):
        assert count_contacts(scene, p, r) == O.oracle_count_contacts(scene, p, r)

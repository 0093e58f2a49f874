"""The native (C++) x-slab driver (csrc/pbdr_slab.cu) on rank-local scenes.

CPU: the rank-local generator reproduces the whole grid's cubes for any
column range (the slab decomposition's premise: local body k is global body
body_first + k, bit-identical), and the slab geometry.
GPU: ranks as threads of this process sharing the one GPU, their halo over
the driver's local hub (the NCCL transport is the same driver with
ncclSend/ncclRecv; this pool gives one GPU per call). Every owned particle
after 45 frames -- through landing, body-body contact and migrations -- equals
the single-handle run of the whole grid bit for bit (refresh = 0), with and
without the boundary/interior overlap; the once-per-substep refresh stays
within the north_star's 1% on the pile aggregates.
"""
import threading

import numpy as np
import pytest

from paper_2603_14634_b200 import pbdr as P
from paper_2603_14634_b200 import slab_native as S


@pytest.mark.parametrize("x_first,x_count", [(0, 16), (0, 5), (5, 6), (11, 5)])
def test_slab_scene_is_a_range_of_the_grid(pbdr, x_first, x_count):
    whole = P.GeneratedScene(5, scale=16)
    assert whole.resamples == 0
    sl = P.GeneratedScene(5, c5_slab=(16, 16, 8, x_first, x_count))
    per = 16 * 8 * 512
    a, b = x_first * per, (x_first + x_count) * per
    assert np.array_equal(sl.positions(), whole.positions()[a:b])
    assert np.array_equal(sl.velocities(), whole.velocities()[a:b])
    assert np.array_equal(sl.array("rest_offsets", 3 * sl.num_particles),
                          whole.array("rest_offsets", 3 * whole.num_particles)[3 * a:3 * b])


def test_slab_spec_geometry():
    s = S.c5_slab_spec(1, 4, columns_per_rank=64)
    assert s.gx == 256 and s.x_first == 61 and s.x_count == 70 and s.body_first == 61 * 64 * 32
    assert list(s.owned_columns) == list(range(64, 128))
    # edges sit halfway between the last column of a slab and the next one
    assert np.isclose(s.edges[1] + 0.1, -0.5 * 0.2 * 255 + 0.2 * 64)
    with pytest.raises(P.ConfigError):
        S.c5_slab_spec(0, 2, ghost_cols=1)


def _run_threads(world, cols, frames, refresh=0, overlap=0):
    hub = P.slab_hub_create(world)
    specs = [S.c5_slab_spec(r, world, columns_per_rank=cols, gy=16, gz=8) for r in range(world)]
    scenes = [S.generate(sp) for sp in specs]
    solvers = [P.GpuSolver(sc.desc, sc.cfg) for sc in scenes]
    for sv, sp in zip(solvers, specs):
        S.attach(sv, sp, refresh=refresh, overlap=overlap, hub=hub)
    errs = [None] * world

    def work(r):
        try:
            solvers[r].slab_start()
            solvers[r].slab_step_frames(frames)
        except BaseException as e:  # noqa: BLE001 -- surfaced below
            errs[r] = e

    ts = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=900)
    for e in errs:
        if e is not None:
            raise e
    out = [S.owned_state(sv, sc, sp) for sv, sc, sp in zip(solvers, scenes, specs)]
    info = [sv.slab_info() for sv in solvers]
    for sv in solvers:
        sv.close()
    P.slab_hub_destroy(hub)
    return out, info


def _whole(cols_total, frames):
    g = P.GeneratedScene(5, c5_slab=(cols_total, 16, 8, 0, cols_total))
    s = P.GpuSolver(g.desc, g.cfg)
    s.step_frames(frames)
    p4, v4 = s.read_f32()
    s.close()
    return p4, v4


@pytest.mark.gpu
@pytest.mark.parametrize("world,overlap", [(2, 0), (2, 1), (4, 0)])
def test_native_slabs_bit_exact(pbdr, world, overlap):
    cols = 16 // world
    frames = 45
    p_ref, v_ref = _whole(16, frames)
    out, info = _run_threads(world, cols, frames, overlap=overlap)
    seen = np.zeros(len(p_ref), bool)
    for ids, slots, p4, v4 in out:
        assert np.array_equal(p4, p_ref[slots]), "owned positions differ from the single-handle run"
        assert np.array_equal(v4, v_ref[slots])
        assert not seen[slots].any(), "a particle owned by two ranks"
        seen[slots] = True
    assert seen.all(), "every body is owned by exactly one rank"
    assert sum(i["ghost_bodies"] for i in info) > 0
    assert all(i["frames"] == frames for i in info)


@pytest.mark.gpu
def test_native_slabs_substep_refresh_aggregates(pbdr):
    frames = 45
    p_ref, v_ref = _whole(16, frames)
    out, _ = _run_threads(2, 8, frames, refresh=1)
    p = np.zeros_like(p_ref)
    v = np.zeros_like(v_ref)
    for ids, slots, p4, v4 in out:
        p[slots], v[slots] = p4, v4
    com, com_ref = p[:, :3].mean(0), p_ref[:, :3].mean(0)
    ke, ke_ref = (v[:, :3] ** 2).sum(), (v_ref[:, :3] ** 2).sum()
    assert np.abs(com - com_ref).max() <= 0.01 * np.abs(com_ref).max()
    assert abs(ke - ke_ref) <= 0.01 * ke_ref


@pytest.mark.gpu
def test_nccl_transport_single_rank(pbdr):
    # The NCCL transport end to end on the one GPU this pool provides: a
    # world-1 communicator (no peers, so no exchange), the driver's per-frame
    # repartition and role set-up on the whole grid; equal to the plain handle.
    frames = 5
    p_ref, v_ref = _whole(16, frames)
    spec = S.c5_slab_spec(0, 1, columns_per_rank=16, gy=16, gz=8)
    g = S.generate(spec)
    s = P.GpuSolver(g.desc, g.cfg)
    S.attach(s, spec, overlap=1, nccl_id=P.nccl_unique_id())
    s.slab_start()
    s.slab_step_frames(frames)
    ids, slots, p4, v4 = S.owned_state(s, g, spec)
    assert len(ids) == g.num_bodies
    assert np.array_equal(p4, p_ref[slots]) and np.array_equal(v4, v_ref[slots])

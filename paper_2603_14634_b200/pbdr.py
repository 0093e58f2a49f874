"""Python host mirror of the reference's solver API over the B200 C-ABI.

The reference's scene/step API is C++ (proj/include/pbdr/scene.hpp:17-82,
body.hpp:11-66, errors.hpp:8-44; step() specified in SPEC.md:326-334). This
module binds include/pbdr_gpu.h with ctypes so tests and bench.py drive the
same entry points a C++ caller (include/pbdr/pbdr_b200.hpp) or a reference-side
binding would. There is no CPU fallback: if the CUDA library is missing, or no
sm_100 device is present, every compute call raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PBDR_LIB_PATH") or os.path.join(_HERE, "lib", "libpbdr_gpu.so")
# Host-only half of the ABI (scene generation, RNG, pack_box, last-error
# state): no CUDA. libpbdr_gpu.so links against it, so both handles see one
# error state; the CPU reference arm loads only this one.
HOST_LIB_PATH = os.environ.get("PBDR_HOST_LIB_PATH") or os.path.join(_HERE, "lib", "libpbdr_host.so")

NBR_CAP = 32
KCLASS_NAMES = ("integrate_key", "sort_histogram", "sort_onesweep", "cell_ranges",
                "neighbours", "iteration", "memset", "broadphase")

# ---- status codes / exceptions (errors.hpp:8-44) ---------------------------
OK, ERR_DEGENERATE, ERR_RANK_DEFICIENT, ERR_EMPTY_PACKING, ERR_INVALID_MOMENT, \
    ERR_CONFIG, ERR_SIMULATION, ERR_CUDA, ERR_GENERIC = range(9)


class Error(RuntimeError):
    """pbdr::Error"""


class DegenerateConfigError(Error):
    pass


class RankDeficientError(Error):
    def __init__(self, msg, axis):
        super().__init__(msg)
        self.axis = tuple(axis)


class EmptyPackingError(Error):
    pass


class InvalidMomentError(Error):
    pass


class ConfigError(Error):
    def __init__(self, msg, key_path):
        super().__init__(msg)
        self.key_path = key_path


class SimulationError(Error):
    def __init__(self, msg, frame_index, body):
        super().__init__(msg)
        self.frame_index = frame_index
        self.body = body


class CudaUnavailableError(Error):
    """No usable sm_100 device or a CUDA failure (no CPU fallback exists)."""


# ---- C structures --------------------------------------------------------------
class SolverCfg(C.Structure):
    _fields_ = [("frame_rate", C.c_double), ("substeps", C.c_int32),
                ("solver_iterations", C.c_int32), ("precision", C.c_int32),
                ("velocity_update", C.c_int32), ("linear_momentum_fix", C.c_int32),
                ("angular_momentum_fix", C.c_int32), ("momentum_frequency", C.c_int32),
                ("backend", C.c_int32), ("gravity", C.c_double)]


class Plane(C.Structure):
    _fields_ = [("point", C.c_double * 3), ("normal", C.c_double * 3), ("friction", C.c_double)]


class ForceProgram(C.Structure):
    _fields_ = [("force", C.c_double * 3), ("torque", C.c_double * 3), ("t_start", C.c_double),
                ("t_stop", C.c_double), ("gravity_exempt", C.c_int32), ("reserved", C.c_int32)]


class SceneDesc(C.Structure):
    _fields_ = [("num_particles", C.c_int64), ("position", C.POINTER(C.c_double)),
                ("velocity", C.POINTER(C.c_double)), ("inv_mass", C.POINTER(C.c_double)),
                ("radius", C.POINTER(C.c_double)), ("body_id", C.POINTER(C.c_int32)),
                ("num_bodies", C.c_int32), ("body_offsets", C.POINTER(C.c_int64)),
                ("body_indices", C.POINTER(C.c_int32)), ("rest_offsets", C.POINTER(C.c_double)),
                ("total_mass", C.POINTER(C.c_double)), ("rest_com", C.POINTER(C.c_double)),
                ("programs", C.POINTER(ForceProgram)), ("ground", Plane),
                ("has_ground", C.c_int32), ("contact_relaxation", C.c_double),
                ("num_walls", C.c_int32), ("walls", C.POINTER(Plane)),
                ("body_scene", C.POINTER(C.c_int32)), ("tile_kp", C.c_int32)]


class SlabConfig(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32), ("edges", C.POINTER(C.c_double)),
                ("ghost_band", C.c_double), ("margin", C.c_double), ("body_first", C.c_int64),
                ("refresh", C.c_int32), ("overlap", C.c_int32)]


class BodyStats(C.Structure):
    _fields_ = [("com", C.c_double * 3), ("quat", C.c_double * 4), ("linear", C.c_double * 3),
                ("angular", C.c_double * 3)]


class Info(C.Structure):
    _fields_ = [("num_particles", C.c_int64), ("num_bodies", C.c_int32), ("num_ctas", C.c_int32),
                ("hash_bits", C.c_int32), ("sort_passes", C.c_int32),
                ("launches_per_frame", C.c_int64), ("device_bytes", C.c_int64),
                ("device", C.c_int32), ("sm_count", C.c_int32), ("cell_size", C.c_float),
                ("dt", C.c_float), ("tile_kp", C.c_int32), ("scene_cluster", C.c_int32)]


_lib = None


FIELD_POSITION, FIELD_VELOCITY, FIELD_ANCHOR, FIELD_ROTATION = 0, 1, 2, 3


def lib() -> C.CDLL:
    """Loads the in-tree CUDA library; raises loudly when it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(the PBD-R path has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        vp, i32, i64, dp, fp = C.c_void_p, C.c_int32, C.c_int64, C.POINTER(C.c_double), C.c_void_p
        L.pbdr_gpu_create.argtypes = [C.POINTER(SceneDesc), C.POINTER(SolverCfg), C.c_int, C.POINTER(vp)]
        L.pbdr_gpu_destroy.argtypes = [vp]
        L.pbdr_gpu_destroy.restype = None
        for name in ("pbdr_gpu_step", "pbdr_gpu_step_frames"):
            getattr(L, name).argtypes = [vp, i64]
        L.pbdr_gpu_read_particles.argtypes = [vp, vp, vp]
        L.pbdr_gpu_write_particles.argtypes = [vp, vp, vp]
        L.pbdr_gpu_read_f32.argtypes = [vp, vp, vp]
        L.pbdr_gpu_write_f32.argtypes = [vp, vp, vp]
        L.pbdr_gpu_write_f32_async.argtypes = [vp, vp, vp]
        L.pbdr_gpu_read_f32_async.argtypes = [vp, vp, vp]
        L.pbdr_gpu_step_frames_async.argtypes = [vp, i64]
        L.pbdr_gpu_read_bodies.argtypes = [vp, vp]
        L.pbdr_nccl_unique_id.argtypes = [vp]
        L.pbdr_gpu_slab_attach_nccl.argtypes = [vp, C.POINTER(SlabConfig), vp]
        L.pbdr_slab_hub_create.argtypes = [C.c_int]
        L.pbdr_slab_hub_create.restype = vp
        L.pbdr_slab_hub_destroy.argtypes = [vp]
        L.pbdr_slab_hub_destroy.restype = None
        L.pbdr_gpu_slab_attach_local.argtypes = [vp, C.POINTER(SlabConfig), vp]
        L.pbdr_gpu_slab_start.argtypes = [vp]
        L.pbdr_gpu_slab_step_frames.argtypes = [vp, i64]
        L.pbdr_gpu_slab_owned.argtypes = [vp, vp, i64, C.POINTER(i64)]
        L.pbdr_gpu_slab_info.argtypes = [vp, vp]
        L.pbdr_gpu_set_time.argtypes = [vp, i64]
        L.pbdr_gpu_get_time.argtypes = [vp, C.POINTER(i64)]
        L.pbdr_gpu_info.argtypes = [vp, C.POINTER(Info)]
        L.pbdr_gpu_time_frames.argtypes = [vp, i64, C.POINTER(C.c_float)]
        L.pbdr_gpu_profile_frames.argtypes = [vp, i64, vp, vp]
        L.pbdr_gpu_debug_prologue.argtypes = [vp]
        L.pbdr_gpu_debug_iteration.argtypes = [vp, C.c_int]
        L.pbdr_gpu_debug_read_keys.argtypes = [vp, vp, vp]
        L.pbdr_gpu_debug_read_sorted.argtypes = [vp, vp, vp]
        L.pbdr_gpu_debug_read_candidates.argtypes = [vp, vp, vp]
        L.pbdr_gpu_debug_read_init.argtypes = [vp, vp]
        L.pbdr_gpu_debug_read_anchor.argtypes = [vp, vp]
        L.pbdr_gpu_debug_write_anchor.argtypes = [vp, vp]
        L.pbdr_gpu_debug_phase_timing.argtypes = [vp, vp]
        L.pbdr_gpu_debug_near_count.argtypes = [vp, C.POINTER(i64)]
        L.pbdr_gpu_debug_read_rquat.argtypes = [vp, vp]
        L.pbdr_gpu_debug_write_rquat.argtypes = [vp, vp]
        for name in ("pbdr_gpu_substep_begin", "pbdr_gpu_substep_iteration", "pbdr_gpu_sync"):
            getattr(L, name).argtypes = [vp]
        L.pbdr_gpu_stream.argtypes = [vp, C.POINTER(vp)]
        L.pbdr_gpu_trajectory_enable.argtypes = [vp, i64]
        L.pbdr_gpu_trajectory_drain.argtypes = [vp, vp, vp, i64, C.POINTER(i64)]
        L.pbdr_gpu_set_roles.argtypes = [vp, vp]
        for name in ("pbdr_gpu_gather", "pbdr_gpu_scatter"):
            getattr(L, name).argtypes = [vp, C.c_int, vp, i64, vp]
        L.pbdr_pack_mesh.argtypes = [vp, C.c_int32, vp, C.c_int32, C.c_double, C.c_int, vp, i64, vp, vp, vp]
        _lib = L
    return _lib


_host = None


def host_lib() -> C.CDLL:
    """Loads the host-only half of the ABI (no CUDA): scene generators,
    splitmix64, pack_box and the last-error state."""
    global _host
    if _host is None:
        if not os.path.exists(HOST_LIB_PATH):
            raise ImportError(f"{HOST_LIB_PATH} is missing: run __graft_entry__.build()")
        L = C.CDLL(HOST_LIB_PATH)
        vp, i32, i64, dp = C.c_void_p, C.c_int32, C.c_int64, C.POINTER(C.c_double)
        L.pbdr_last_error.restype = C.c_char_p
        L.pbdr_last_error_key.restype = C.c_char_p
        L.pbdr_last_error_payload.argtypes = [dp, C.POINTER(i64), C.POINTER(i32)]
        L.pbdr_scene_generate.argtypes = [C.c_int, C.c_uint64, i64, C.POINTER(vp)]
        L.pbdr_scene_generate_c4_shard.argtypes = [C.c_uint64, i64, i64, C.POINTER(vp)]
        L.pbdr_scene_generate_c5_slab.argtypes = [C.c_uint64, i64, i64, i64, i64, i64, C.POINTER(vp)]
        L.pbdr_scene_resamples.argtypes = [vp]
        L.pbdr_scene_resamples.restype = i64
        L.pbdr_scene_view.argtypes = [vp, C.POINTER(SceneDesc), C.POINTER(SolverCfg)]
        L.pbdr_scene_frames.argtypes = [vp]
        L.pbdr_scene_frames.restype = i64
        L.pbdr_scene_forced_overlaps.argtypes = [vp]
        L.pbdr_scene_forced_overlaps.restype = i64
        L.pbdr_scene_free.argtypes = [vp]
        L.pbdr_scene_free.restype = None
        L.pbdr_pack_box.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int, vp, vp]
        L.pbdr_rng_u64.argtypes = [C.c_uint64, C.c_int, vp]
        L.pbdr_rng_u64.restype = None
        L.pbdr_rng_unit.argtypes = [C.c_uint64, C.c_int, vp]
        L.pbdr_rng_unit.restype = None
        _host = L
    return _host


def raise_status(status: int):
    """Maps a C-ABI status to the matching pbdr exception (errors.hpp:8-44)."""
    if status == OK:
        return
    L = host_lib()
    msg = L.pbdr_last_error().decode(errors="replace")
    axis = (C.c_double * 3)()
    frame = C.c_int64()
    body = C.c_int32()
    L.pbdr_last_error_payload(axis, C.byref(frame), C.byref(body))
    if status == ERR_DEGENERATE:
        raise DegenerateConfigError(msg)
    if status == ERR_RANK_DEFICIENT:
        raise RankDeficientError(msg, list(axis))
    if status == ERR_EMPTY_PACKING:
        raise EmptyPackingError(msg)
    if status == ERR_INVALID_MOMENT:
        raise InvalidMomentError(msg)
    if status == ERR_CONFIG:
        raise ConfigError(msg, L.pbdr_last_error_key().decode())
    if status == ERR_SIMULATION:
        raise SimulationError(msg, frame.value, body.value)
    if status == ERR_CUDA:
        raise CudaUnavailableError(msg)
    raise Error(msg)


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# ---- solver config ---------------------------------------------------------------
def solver_cfg(frame_rate=100.0, substeps=10, solver_iterations=10, precision=0,
               velocity_update=1, linear_momentum_fix=True, angular_momentum_fix=True,
               momentum_frequency=0, gravity=9.81, backend=1) -> SolverCfg:
    """SolverConfig defaults of scene.hpp:17-28 (pbdr() preset)."""
    return SolverCfg(frame_rate, substeps, solver_iterations, precision, velocity_update,
                     int(linear_momentum_fix), int(angular_momentum_fix), momentum_frequency,
                     backend, gravity)


def pbd_cfg(**kw) -> SolverCfg:
    """SolverConfig::pbd(): legacy velocity update, no momentum fixes (scene.hpp:33-39)."""
    c = solver_cfg(**kw)
    c.velocity_update = 0
    c.linear_momentum_fix = 0
    c.angular_momentum_fix = 0
    return c


# ---- scenes ----------------------------------------------------------------------
class ArrayScene:
    """Owns numpy arrays behind a SceneDesc (a reference Scene as plain arrays)."""

    def __init__(self, position, velocity, inv_mass, radius, body_offsets, rest_offsets,
                 total_mass, rest_com, body_indices=None, body_id=None, ground=None,
                 has_ground=True, contact_relaxation=1.0, walls=(), body_scene=None,
                 programs=None, tile_kp=0):
        n = len(inv_mass)
        nb = len(total_mass)
        self.position = np.ascontiguousarray(position, dtype=np.float64).reshape(n, 3)
        self.velocity = np.ascontiguousarray(velocity, dtype=np.float64).reshape(n, 3)
        self.inv_mass = np.ascontiguousarray(inv_mass, dtype=np.float64)
        self.radius = np.ascontiguousarray(radius, dtype=np.float64)
        self.body_offsets = np.ascontiguousarray(body_offsets, dtype=np.int64)
        self.body_indices = (np.arange(n, dtype=np.int32) if body_indices is None
                             else np.ascontiguousarray(body_indices, dtype=np.int32))
        if body_id is None:
            body_id = np.zeros(n, dtype=np.int32)
            for b in range(nb):
                body_id[self.body_indices[self.body_offsets[b]:self.body_offsets[b + 1]]] = b
        self.body_id = np.ascontiguousarray(body_id, dtype=np.int32)
        self.rest_offsets = np.ascontiguousarray(rest_offsets, dtype=np.float64).reshape(-1, 3)
        self.total_mass = np.ascontiguousarray(total_mass, dtype=np.float64)
        self.rest_com = np.ascontiguousarray(rest_com, dtype=np.float64).reshape(nb, 3)
        self.walls = (Plane * max(1, len(walls)))(*walls) if walls else None
        self.body_scene = None if body_scene is None else np.ascontiguousarray(body_scene, dtype=np.int32)
        self.programs = None if programs is None else (ForceProgram * nb)(*programs)
        d = SceneDesc()
        d.num_particles = n
        d.position = self.position.ctypes.data_as(C.POINTER(C.c_double))
        d.velocity = self.velocity.ctypes.data_as(C.POINTER(C.c_double))
        d.inv_mass = self.inv_mass.ctypes.data_as(C.POINTER(C.c_double))
        d.radius = self.radius.ctypes.data_as(C.POINTER(C.c_double))
        d.body_id = self.body_id.ctypes.data_as(C.POINTER(C.c_int32))
        d.num_bodies = nb
        d.body_offsets = self.body_offsets.ctypes.data_as(C.POINTER(C.c_int64))
        d.body_indices = self.body_indices.ctypes.data_as(C.POINTER(C.c_int32))
        d.rest_offsets = self.rest_offsets.ctypes.data_as(C.POINTER(C.c_double))
        d.total_mass = self.total_mass.ctypes.data_as(C.POINTER(C.c_double))
        d.rest_com = self.rest_com.ctypes.data_as(C.POINTER(C.c_double))
        if self.programs is not None:
            d.programs = C.cast(self.programs, C.POINTER(ForceProgram))
        d.ground = ground if ground is not None else Plane((0, 0, 0), (0, 0, 1), 0.0)
        d.has_ground = int(has_ground)
        d.contact_relaxation = contact_relaxation
        d.num_walls = len(walls)
        if self.walls is not None:
            d.walls = C.cast(self.walls, C.POINTER(Plane))
        if self.body_scene is not None:
            d.body_scene = self.body_scene.ctypes.data_as(C.POINTER(C.c_int32))
        d.tile_kp = tile_kp
        self.desc = d

    @property
    def num_particles(self):
        return len(self.inv_mass)

    @property
    def num_bodies(self):
        return len(self.total_mass)


def rigid_body_arrays(centers_list, radius, masses, velocities=None):
    """Builds ArrayScene inputs for bodies given placed particle centres
    (rest pose = placed pose, uniform mass M/N: add_packed_body semantics)."""
    pos, vel, inv, rad, offs, rest, tm, rc = [], [], [], [], [0], [], [], []
    for b, cen in enumerate(centers_list):
        cen = np.asarray(cen, dtype=np.float64).reshape(-1, 3)
        n = len(cen)
        m = masses[b]
        w = n / m
        mp = np.full(n, 1.0 / w)
        com = (cen * mp[:, None]).sum(0) / mp.sum()
        pos.append(cen)
        vel.append(np.zeros_like(cen) if velocities is None else np.asarray(velocities[b], dtype=np.float64).reshape(-1, 3))
        inv.append(np.full(n, w))
        rad.append(np.full(n, radius))
        offs.append(offs[-1] + n)
        rest.append(cen - com)
        tm.append(mp.sum())
        rc.append(com)
    return dict(position=np.concatenate(pos), velocity=np.concatenate(vel),
                inv_mass=np.concatenate(inv), radius=np.concatenate(rad),
                body_offsets=np.array(offs, dtype=np.int64), rest_offsets=np.concatenate(rest),
                total_mass=np.array(tm), rest_com=np.array(rc))


def scene_with_programs(src, programs) -> "ArrayScene":
    """Copy of a scene (GeneratedScene or ArrayScene) with per-body ForcePrograms
    attached (scene.hpp:53-61: Scene::programs, one per body)."""
    d = src.desc
    n, nb = int(d.num_particles), int(d.num_bodies)

    def arr(name, count, dtype=np.float64):
        ptr = getattr(d, name)
        return np.ctypeslib.as_array(ptr, shape=(count,)).astype(dtype, copy=True) if count else np.zeros(0, dtype)

    walls = [d.walls[i] for i in range(d.num_walls)] if d.num_walls else ()
    body_scene = arr("body_scene", nb, np.int32) if bool(d.body_scene) else None
    return ArrayScene(position=arr("position", 3 * n), velocity=arr("velocity", 3 * n),
                      inv_mass=arr("inv_mass", n), radius=arr("radius", n),
                      body_offsets=arr("body_offsets", nb + 1, np.int64),
                      rest_offsets=arr("rest_offsets", 3 * n), total_mass=arr("total_mass", nb),
                      rest_com=arr("rest_com", 3 * nb), body_indices=arr("body_indices", n, np.int32),
                      body_id=arr("body_id", n, np.int32), ground=d.ground, has_ground=bool(d.has_ground),
                      contact_relaxation=d.contact_relaxation, walls=walls, body_scene=body_scene,
                      programs=list(programs), tile_kp=d.tile_kp)


class GeneratedScene:
    """One of the five BASELINE.json configs, built by the host generator
    (libpbdr_host.so: no CUDA, so the CPU arms can use it too)."""

    def __init__(self, config_id: int, seed: int = 0, scale: int = 0, c4_first_scene: int | None = None,
                 c5_slab: tuple | None = None):
        """c5_slab = (gx, gy, gz, x_first, x_count): config 5's cubes in those
        x-columns of a gx * gy * gz grid (a rank-local slab scene)."""
        L = host_lib()
        h = C.c_void_p()
        if c5_slab is not None:
            st = L.pbdr_scene_generate_c5_slab(seed, *[int(v) for v in c5_slab], C.byref(h))
        elif c4_first_scene is None:
            st = L.pbdr_scene_generate(config_id, seed, scale, C.byref(h))
        else:
            st = L.pbdr_scene_generate_c4_shard(seed, scale, c4_first_scene, C.byref(h))
        raise_status(st)
        self._h = h
        self.config_id = config_id
        self.desc = SceneDesc()
        self.cfg = SolverCfg()
        raise_status(L.pbdr_scene_view(h, C.byref(self.desc), C.byref(self.cfg)))
        self.frames = L.pbdr_scene_frames(h)
        self.forced_overlaps = L.pbdr_scene_forced_overlaps(h)
        self.resamples = L.pbdr_scene_resamples(h)

    @property
    def num_particles(self):
        return self.desc.num_particles

    @property
    def num_bodies(self):
        return self.desc.num_bodies

    def array(self, name, count, dtype=np.float64):
        ptr = getattr(self.desc, name)
        return np.ctypeslib.as_array(ptr, shape=(count,)).astype(dtype, copy=True) if count else np.zeros(0, dtype)

    def positions(self):
        return self.array("position", 3 * self.num_particles).reshape(-1, 3)

    def velocities(self):
        return self.array("velocity", 3 * self.num_particles).reshape(-1, 3)

    def body_offsets(self):
        return self.array("body_offsets", self.num_bodies + 1, np.int64)

    def close(self):
        if getattr(self, "_h", None):
            host_lib().pbdr_scene_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---- solver handle ------------------------------------------------------------------
class GpuSolver:
    """One scene resident on one B200 (pbdr_handle)."""

    def __init__(self, desc: SceneDesc, cfg: SolverCfg, device: int = 0):
        L = lib()
        h = C.c_void_p()
        raise_status(L.pbdr_gpu_create(C.byref(desc), C.byref(cfg), device, C.byref(h)))
        self._h = h
        self.info = Info()
        raise_status(L.pbdr_gpu_info(h, C.byref(self.info)))
        self.n = self.info.num_particles
        self.nb = self.info.num_bodies

    def close(self):
        if getattr(self, "_h", None):
            lib().pbdr_gpu_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def step(self, substeps: int = 1):
        raise_status(lib().pbdr_gpu_step(self._h, substeps))

    def step_frames(self, frames: int = 1):
        raise_status(lib().pbdr_gpu_step_frames(self._h, frames))

    # ---- trajectory emission ------------------------------------
    def enable_trajectory(self, capacity_frames: int):
        self._traj_cap = capacity_frames
        raise_status(lib().pbdr_gpu_trajectory_enable(self._h, capacity_frames))

    def drain_trajectory(self):
        """(t[frames], stats[frames, num_bodies, 13]) of the frames since the last drain."""
        cap = getattr(self, "_traj_cap", 0)
        out = np.zeros((cap, self.nb, 13), np.float64)
        t = np.zeros(cap, np.float64)
        k = C.c_int64()
        raise_status(lib().pbdr_gpu_trajectory_drain(self._h, _ptr(out), _ptr(t), cap, C.byref(k)))
        return t[:k.value].copy(), out[:k.value].copy()

    # ---- staged stepping / x-slab decomposition (include/pbdr_gpu.h) ----------
    def substep_begin(self):
        raise_status(lib().pbdr_gpu_substep_begin(self._h))

    def substep_iteration(self):
        raise_status(lib().pbdr_gpu_substep_iteration(self._h))

    def sync(self):
        raise_status(lib().pbdr_gpu_sync(self._h))

    def stream_handle(self) -> int:
        s = C.c_void_p()
        raise_status(lib().pbdr_gpu_stream(self._h, C.byref(s)))
        return s.value or 0

    def set_roles(self, roles=None):
        r = None if roles is None else np.ascontiguousarray(roles, np.int8)
        raise_status(lib().pbdr_gpu_set_roles(self._h, None if r is None else r.ctypes.data_as(C.c_void_p)))

    def gather_dev(self, field: int, index_ptr: int, count: int, dst_ptr: int):
        """float4 records by index, device pointers, enqueued on the handle's stream."""
        raise_status(lib().pbdr_gpu_gather(self._h, field, C.c_void_p(index_ptr), count, C.c_void_p(dst_ptr)))

    def scatter_dev(self, field: int, index_ptr: int, count: int, src_ptr: int):
        raise_status(lib().pbdr_gpu_scatter(self._h, field, C.c_void_p(index_ptr), count, C.c_void_p(src_ptr)))

    def time_frames(self, frames: int) -> float:
        ms = C.c_float()
        raise_status(lib().pbdr_gpu_time_frames(self._h, frames, C.byref(ms)))
        return ms.value

    def profile_frames(self, frames: int):
        ms = np.zeros(len(KCLASS_NAMES), dtype=np.float32)
        launches = np.zeros(len(KCLASS_NAMES), dtype=np.int64)
        raise_status(lib().pbdr_gpu_profile_frames(self._h, frames, _ptr(ms), _ptr(launches)))
        return {k: (float(ms[i]), int(launches[i])) for i, k in enumerate(KCLASS_NAMES)}

    def read_f32(self, out_pos=None, out_vel=None):
        p = np.empty((self.n, 4), np.float32) if out_pos is None else out_pos
        v = np.empty((self.n, 4), np.float32) if out_vel is None else out_vel
        raise_status(lib().pbdr_gpu_read_f32(self._h, _ptr(p), _ptr(v)))
        return p, v

    def write_f32(self, pos4=None, vel4=None):
        raise_status(lib().pbdr_gpu_write_f32(self._h, _ptr(pos4), _ptr(vel4)))

    # asynchronous (pinned buffers; completion and errors at sync())
    def write_f32_async(self, pos4=None, vel4=None):
        raise_status(lib().pbdr_gpu_write_f32_async(self._h, _ptr(pos4), _ptr(vel4)))

    def read_f32_async(self, pos4=None, vel4=None):
        raise_status(lib().pbdr_gpu_read_f32_async(self._h, _ptr(pos4), _ptr(vel4)))

    def step_frames_async(self, frames: int = 1):
        raise_status(lib().pbdr_gpu_step_frames_async(self._h, frames))

    def read_particles(self):
        p = np.empty((self.n, 3), np.float64)
        v = np.empty((self.n, 3), np.float64)
        raise_status(lib().pbdr_gpu_read_particles(self._h, _ptr(p), _ptr(v)))
        return p, v

    def write_particles(self, pos=None, vel=None):
        pos = None if pos is None else np.ascontiguousarray(pos, np.float64)
        vel = None if vel is None else np.ascontiguousarray(vel, np.float64)
        raise_status(lib().pbdr_gpu_write_particles(self._h, _ptr(pos), _ptr(vel)))

    # ---- native x-slab decomposition (pbdr_gpu_slab_*) ------------------------
    def slab_attach(self, rank, world, edges, ghost_band, margin, body_first, refresh=0, overlap=0,
                    hub=None, nccl_id: bytes | None = None):
        """Attach the C++ slab driver: over a local hub (thread ranks sharing
        this GPU) or over NCCL (nccl_id: 128 bytes from nccl_unique_id())."""
        self._slab_edges = (C.c_double * len(edges))(*[float(e) for e in edges])
        cfg = SlabConfig(rank, world, C.cast(self._slab_edges, C.POINTER(C.c_double)), ghost_band, margin,
                         body_first, refresh, overlap)
        self._slab_cfg = cfg
        if hub is not None:
            raise_status(lib().pbdr_gpu_slab_attach_local(self._h, C.byref(cfg), C.c_void_p(hub)))
        else:
            buf = (C.c_uint8 * 128).from_buffer_copy(nccl_id)
            raise_status(lib().pbdr_gpu_slab_attach_nccl(self._h, C.byref(cfg), buf))

    def slab_start(self):
        raise_status(lib().pbdr_gpu_slab_start(self._h))

    def slab_step_frames(self, frames: int = 1):
        raise_status(lib().pbdr_gpu_slab_step_frames(self._h, frames))

    def slab_owned(self) -> np.ndarray:
        n = C.c_int64()
        raise_status(lib().pbdr_gpu_slab_owned(self._h, None, 0, C.byref(n)))
        out = np.empty(n.value, np.int32)
        raise_status(lib().pbdr_gpu_slab_owned(self._h, _ptr(out), n.value, C.byref(n)))
        return out

    def slab_info(self) -> dict:
        out = np.zeros(6, np.int64)
        raise_status(lib().pbdr_gpu_slab_info(self._h, _ptr(out)))
        keys = ("owned_bodies", "owned_particles", "ghost_bodies", "halo_bytes_per_iteration", "migrations", "frames")
        return {k: int(v) for k, v in zip(keys, out)}

    def set_time(self, substep: int):
        """Simulation time as a substep index (ForceProgram windows, error frames)."""
        raise_status(lib().pbdr_gpu_set_time(self._h, substep))

    def get_time(self) -> int:
        t = C.c_int64()
        raise_status(lib().pbdr_gpu_get_time(self._h, C.byref(t)))
        return t.value

    def read_bodies(self):
        out = np.zeros((self.nb, 13), np.float64)
        raise_status(lib().pbdr_gpu_read_bodies(self._h, _ptr(out)))
        return out  # com[0:3], quat[3:7], P[7:10], L[10:13]

    # -- replay hooks ---------------------------------------------------------
    def debug_prologue(self):
        raise_status(lib().pbdr_gpu_debug_prologue(self._h))

    def debug_iteration(self):
        raise_status(lib().pbdr_gpu_debug_iteration(self._h, 0))

    def debug_keys(self):
        hsh = np.empty(self.n, np.uint32)
        cell = np.empty((self.n, 3), np.int32)
        raise_status(lib().pbdr_gpu_debug_read_keys(self._h, _ptr(hsh), _ptr(cell)))
        return hsh, cell

    def debug_sorted(self):
        """Sorted (key, slot) pairs of the broadphase-filtered particles."""
        k = np.empty(self.n, np.uint32)
        v = np.empty(self.n, np.uint32)
        raise_status(lib().pbdr_gpu_debug_read_sorted(self._h, _ptr(k), _ptr(v)))
        m = C.c_int64()
        raise_status(lib().pbdr_gpu_debug_near_count(self._h, C.byref(m)))
        return k[:m.value], v[:m.value]

    def debug_candidates(self):
        c = np.empty(self.n, np.int32)
        lst = np.empty((self.n, NBR_CAP), np.int32)
        raise_status(lib().pbdr_gpu_debug_read_candidates(self._h, _ptr(c), _ptr(lst)))
        return c, lst

    def debug_init(self):
        x = np.empty((self.n, 4), np.float32)
        raise_status(lib().pbdr_gpu_debug_read_init(self._h, _ptr(x)))
        return x

    def debug_anchor(self):
        a = np.empty((self.nb, 3), np.float32)
        raise_status(lib().pbdr_gpu_debug_read_anchor(self._h, _ptr(a)))
        return a

    def debug_phase_timing(self):
        """clock64 stamps per CTA of one iteration launch (see pbdr_gpu.h)."""
        out = np.zeros((self.info.num_ctas, 16), np.int64)
        raise_status(lib().pbdr_gpu_debug_phase_timing(self._h, _ptr(out)))
        return out

    def debug_rquat(self):
        q = np.empty((self.nb, 4), np.float32)
        raise_status(lib().pbdr_gpu_debug_read_rquat(self._h, _ptr(q)))
        return q

    def debug_write_rquat(self, q):
        q = np.ascontiguousarray(q, np.float32)
        raise_status(lib().pbdr_gpu_debug_write_rquat(self._h, _ptr(q)))

    def debug_write_anchor(self, a):
        a = np.ascontiguousarray(a, np.float32)
        raise_status(lib().pbdr_gpu_debug_write_anchor(self._h, _ptr(a)))


def pack_box(half_extents, n):
    """geometry.cpp:32-55 pack_box through the library's host helper."""
    c = np.empty((n ** 3, 3), np.float64)
    r = C.c_double()
    raise_status(host_lib().pbdr_pack_box(half_extents[0], half_extents[1], half_extents[2], n, _ptr(c), C.byref(r)))
    return c, r.value


def pack_mesh(vertices, triangles, radius, device: int = 0):
    """GPU pack_mesh (geometry.cpp:151-195): grid points inside the closed
    triangle mesh, in grid order. Returns (centers[k, 3], candidates, ambiguous)."""
    v = np.ascontiguousarray(vertices, np.float64).reshape(-1, 3)
    t = np.ascontiguousarray(triangles, np.int32).reshape(-1, 3)
    L = lib()
    cnt, cand, amb = C.c_int64(), C.c_int64(), C.c_int64()
    raise_status(L.pbdr_pack_mesh(_ptr(v), len(v), _ptr(t), len(t), radius, device, None, 0,
                                  C.byref(cnt), C.byref(cand), C.byref(amb)))
    out = np.empty((cnt.value, 3), np.float64)
    raise_status(L.pbdr_pack_mesh(_ptr(v), len(v), _ptr(t), len(t), radius, device, _ptr(out), cnt.value,
                                  C.byref(cnt), C.byref(cand), C.byref(amb)))
    return out, cand.value, amb.value


def rng_u64(seed, count):
    out = np.empty(count, np.uint64)
    host_lib().pbdr_rng_u64(seed, count, _ptr(out))
    return out


def rng_unit(seed, count):
    out = np.empty(count, np.float64)
    host_lib().pbdr_rng_unit(seed, count, _ptr(out))
    return out


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    raise_status(lib().pbdr_nccl_unique_id(buf))
    return bytes(buf)


def slab_hub_create(world: int) -> int:
    """Local hub for `world` thread ranks sharing one GPU (pbdr_slab_hub_create)."""
    h = lib().pbdr_slab_hub_create(world)
    if not h:
        raise Error("pbdr_slab_hub_create failed")
    return h


def slab_hub_destroy(hub: int):
    lib().pbdr_slab_hub_destroy(C.c_void_p(hub))


def cuda_device_count() -> int:
    try:
        cudart = C.CDLL("libcudart.so.12")
    except OSError:
        return 0
    n = C.c_int(0)
    if cudart.cudaGetDeviceCount(C.byref(n)) != 0:
        return 0
    return n.value


@dataclass
class Workload:
    config_id: int
    name: str
    seed: int = 0
    scale: int = 0


CONFIG_NAMES = {1: "c1_single_cube_512", 2: "c2_pile_64_cubes", 3: "c3_large_pile_8192_bodies",
                4: "c4_batched_4096_scenes", 5: "c5_giant_scene_131072_cubes"}

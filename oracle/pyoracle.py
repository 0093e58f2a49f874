"""TEST INFRASTRUCTURE ONLY: ctypes binding of the CPU oracle
(oracle/build/liboracle.so, a restatement of the reference's PBD-R step — see
the header of oracle/pbdr_oracle.cpp) and of the reference's own compiled
math/body/geometry (oracle/_ref/libpbdr_ref.so, built only where
/root/reference exists).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import
this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_PATH = os.path.join(HERE, "build", "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libpbdr_ref.so")
NBR_CAP = 32

_olib = None
_rlib = None


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def olib():
    global _olib
    if _olib is None:
        if not os.path.exists(ORACLE_PATH):
            raise ImportError(f"{ORACLE_PATH} missing: run `make -C oracle`")
        L = C.CDLL(ORACLE_PATH)
        vp = C.c_void_p
        L.oracle_create.argtypes = [vp, vp, C.c_int, C.POINTER(vp)]
        L.oracle_destroy.argtypes = [vp]
        L.oracle_destroy.restype = None
        for name in ("oracle_integrate", "oracle_candidates", "oracle_iteration", "oracle_end_substep"):
            getattr(L, name).argtypes = [vp]
            getattr(L, name).restype = None
        L.oracle_step.argtypes = [vp, C.c_int64]
        L.oracle_error.argtypes = [vp, vp, vp, vp]
        for name in ("oracle_read_f32", "oracle_write_f32", "oracle_read_particles",
                     "oracle_read_keys", "oracle_read_candidates"):
            getattr(L, name).argtypes = [vp, vp, vp]
            getattr(L, name).restype = None
        for name in ("oracle_read_init", "oracle_write_init", "oracle_read_anchor",
                     "oracle_write_anchor", "oracle_body_stats", "oracle_read_rquat", "oracle_write_rquat"):
            getattr(L, name).argtypes = [vp, vp]
            getattr(L, name).restype = None
        L.oracle_num_slots.argtypes = [vp]
        L.oracle_num_slots.restype = C.c_int64
        L.oracle_tile_kp.argtypes = [vp]
        L.oracle_tile_kp.restype = C.c_int
        L.oracle_pack_mesh.argtypes = [vp, C.c_int, vp, C.c_int, C.c_double, vp, C.c_long, vp, vp, vp]
        L.oracle_set_roles.argtypes = [vp, vp]
        L.oracle_set_roles.restype = None
        for name in ("oracle_gather", "oracle_scatter"):
            getattr(L, name).argtypes = [vp, C.c_int, vp, C.c_int64, vp]
            getattr(L, name).restype = None
        L.oracle_cell_size.argtypes = [vp]
        L.oracle_cell_size.restype = C.c_float
        L.oracle_polar.argtypes = [vp, vp, vp]
        L.oracle_polar_warm.argtypes = [vp, vp, vp, vp]
        L.oracle_sym_eigen.argtypes = [vp, vp, vp]
        L.oracle_sym_eigen.restype = None
        L.oracle_inertia_solve.argtypes = [vp, vp, vp, vp]
        L.oracle_inertia_solve.restype = C.c_uint
        L.oracle_kat_ground.argtypes = [vp, vp, C.c_float, C.c_int, vp, C.c_float, vp]
        L.oracle_kat_ground.restype = None
        L.oracle_kat_pp.argtypes = [vp, C.c_float, C.c_int64, vp, C.c_float, C.c_int64, C.c_float, C.c_float, vp]
        L.oracle_kat_pp.restype = None
        L.oracle_kat_body_iteration.argtypes = [C.c_int, vp, vp, vp, vp, vp, vp, vp, C.c_float, C.c_float,
                                                C.c_int, C.c_int, C.c_int, vp, vp]
        L.oracle_kat_body_iteration.restype = C.c_uint
        L.oracle_kat_momentum.argtypes = [C.c_int, vp, vp, vp, vp, vp, C.c_float, C.c_int, C.c_int, vp, vp, vp]
        L.oracle_kat_momentum.restype = C.c_uint
        L.o64_create.argtypes = [vp, vp, C.c_int, C.POINTER(vp)]
        L.o64_destroy.argtypes = [vp]
        L.o64_destroy.restype = None
        L.o64_step.argtypes = [vp, C.c_int64]
        for name in ("o64_read", "o64_write"):
            getattr(L, name).argtypes = [vp, vp, vp]
            getattr(L, name).restype = None
        L.o64_body_stats.argtypes = [vp, vp]
        L.o64_body_stats.restype = None
        L.o64_error.argtypes = [vp, vp, vp, vp]
        _olib = L
    return _olib


def _bind_ref_api(L):
    vp = C.c_void_p
    L.ref_rng_u64.argtypes = [C.c_uint64, C.c_int, vp]
    L.ref_pack_mesh.argtypes = [vp, C.c_int, vp, C.c_int, C.c_double, vp, C.c_long, vp, vp, vp]
    L.ref_rng_u64.restype = None
    L.ref_rng_unit.argtypes = [C.c_uint64, C.c_int, vp]
    L.ref_rng_unit.restype = None
    L.ref_pack_box.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int, vp, vp]
    L.ref_polar.argtypes = [vp, vp, vp, vp, C.c_double]
    L.ref_sym_eigen.argtypes = [vp, vp, vp]
    L.ref_invert_spd.argtypes = [vp, vp, vp]
    L.ref_pseudo_invert_spd.argtypes = [vp, vp, vp, vp]
    L.ref_inverse.argtypes = [vp, vp]
    L.ref_body_props.argtypes = [C.c_int, vp, vp, vp, vp, vp, vp, vp, vp, vp]
    L.ref_extract_pose.argtypes = [C.c_int, vp, vp, vp, vp, vp]
    L.ref_distribute_wrench.argtypes = [C.c_int, vp, vp, vp, vp, vp, vp]
    L.ref_geodesic_deg.argtypes = [vp, vp]
    L.ref_geodesic_deg.restype = C.c_double
    L.ref_unwrapped_deg.argtypes = [vp, vp]
    L.ref_unwrapped_deg.restype = C.c_double
    L.ref_quat_to_matrix.argtypes = [vp, vp]
    L.ref_quat_to_matrix.restype = None
    L.ref_matrix_to_quat.argtypes = [vp, vp]
    L.ref_matrix_to_quat.restype = None
    return L


def rlib():
    """The reference's own math/body/geometry (oracle/_ref); None when not built."""
    global _rlib
    if _rlib is None:
        if not os.path.exists(REF_PATH):
            return None
        _rlib = _bind_ref_api(C.CDLL(REF_PATH))
    return _rlib


def ref_api(path):
    """ref_shim.cpp's extern "C" functions from any build of it: the
    reference's own code (oracle/_ref) or the product's drop-in headers and
    libraries (build/libdropin_shim.so)."""
    return _bind_ref_api(C.CDLL(path))


class Oracle:
    """CPU restatement of the substep loop on one scene (SceneDesc from the
    product's pbdr module, so both arms see identical inputs)."""

    def __init__(self, desc, cfg, threads: int = 0):
        L = olib()
        if threads <= 0:
            threads = os.cpu_count() or 1
        h = C.c_void_p()
        st = L.oracle_create(C.addressof(desc), C.addressof(cfg), threads, C.byref(h))
        if st != 0:
            raise RuntimeError(f"oracle_create failed with status {st}")
        self._h = h
        self.n = L.oracle_num_slots(h)
        self.nb = desc.num_bodies
        self.threads = threads

    def close(self):
        if getattr(self, "_h", None):
            olib().oracle_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def step(self, substeps=1) -> int:
        return olib().oracle_step(self._h, substeps)

    def integrate(self):
        olib().oracle_integrate(self._h)

    def candidates(self):
        olib().oracle_candidates(self._h)

    def iteration(self):
        olib().oracle_iteration(self._h)

    def end_substep(self):
        olib().oracle_end_substep(self._h)

    # ---- slab decomposition (mirrors GpuSolver.set_roles / gather / scatter) --
    def set_roles(self, roles=None):
        r = None if roles is None else np.ascontiguousarray(roles, np.int8)
        olib().oracle_set_roles(self._h, _p(r))

    def gather(self, field, index):
        index = np.ascontiguousarray(index, np.int32)
        out = np.empty((len(index), 4), np.float32)
        olib().oracle_gather(self._h, field, _p(index), len(index), _p(out))
        return out

    def scatter(self, field, index, values):
        index = np.ascontiguousarray(index, np.int32)
        values = np.ascontiguousarray(values, np.float32).reshape(len(index), 4)
        olib().oracle_scatter(self._h, field, _p(index), len(index), _p(values))

    def error(self):
        bits = C.c_uint32()
        body = C.c_int32()
        axis = np.zeros(3)
        st = olib().oracle_error(self._h, C.byref(bits), C.byref(body), _p(axis))
        return st, bits.value, body.value, axis

    def read_f32(self):
        p = np.empty((self.n, 4), np.float32)
        v = np.empty((self.n, 4), np.float32)
        olib().oracle_read_f32(self._h, _p(p), _p(v))
        return p, v

    def write_f32(self, pos4=None, vel4=None):
        pos4 = None if pos4 is None else np.ascontiguousarray(pos4, np.float32)
        vel4 = None if vel4 is None else np.ascontiguousarray(vel4, np.float32)
        olib().oracle_write_f32(self._h, _p(pos4), _p(vel4))

    def read_init(self):
        x = np.empty((self.n, 4), np.float32)
        olib().oracle_read_init(self._h, _p(x))
        return x

    def write_init(self, x):
        olib().oracle_write_init(self._h, _p(np.ascontiguousarray(x, np.float32)))

    def read_anchor(self):
        a = np.empty((self.nb, 3), np.float32)
        olib().oracle_read_anchor(self._h, _p(a))
        return a

    def write_anchor(self, a):
        olib().oracle_write_anchor(self._h, _p(np.ascontiguousarray(a, np.float32)))

    def read_rquat(self):
        q = np.empty((self.nb, 4), np.float32)
        olib().oracle_read_rquat(self._h, _p(q))
        return q

    def write_rquat(self, q):
        olib().oracle_write_rquat(self._h, _p(np.ascontiguousarray(q, np.float32)))

    def read_particles(self):
        p = np.empty((self.n, 3))
        v = np.empty((self.n, 3))
        olib().oracle_read_particles(self._h, _p(p), _p(v))
        return p, v

    def keys(self):
        h = np.empty(self.n, np.uint32)
        c = np.empty((self.n, 3), np.int32)
        olib().oracle_read_keys(self._h, _p(h), _p(c))
        return h, c

    def read_candidates(self):
        c = np.empty(self.n, np.int32)
        lst = np.empty((self.n, NBR_CAP), np.int32)
        olib().oracle_read_candidates(self._h, _p(c), _p(lst))
        return c, lst

    def body_stats(self):
        out = np.zeros((self.nb, 13))
        olib().oracle_body_stats(self._h, _p(out))
        return out

    @property
    def tile_kp(self):
        return olib().oracle_tile_kp(self._h)

    @property
    def cell_size(self):
        return olib().oracle_cell_size(self._h)


class Oracle64:
    """The independent fp64 restatement (oracle/pbdr_oracle64.cpp): plain
    fp64 body sums, the reference's cold scaled-Newton polar and SPD
    pseudo-inverse, caller particle order. Compared with the GPU at the
    north_star tolerances, never bit for bit."""

    def __init__(self, desc, cfg, threads: int = 0):
        L = olib()
        if threads <= 0:
            threads = os.cpu_count() or 1
        h = C.c_void_p()
        st = L.o64_create(C.addressof(desc), C.addressof(cfg), threads, C.byref(h))
        if st != 0:
            raise RuntimeError(f"o64_create failed with status {st}")
        self._h = h
        self.n = desc.num_particles
        self.nb = desc.num_bodies

    def close(self):
        if getattr(self, "_h", None):
            olib().o64_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def step(self, substeps=1) -> int:
        return olib().o64_step(self._h, substeps)

    def read_particles(self):
        p = np.empty((self.n, 3))
        v = np.empty((self.n, 3))
        olib().o64_read(self._h, _p(p), _p(v))
        return p, v

    def write_particles(self, pos=None, vel=None):
        pos = None if pos is None else np.ascontiguousarray(pos, np.float64)
        vel = None if vel is None else np.ascontiguousarray(vel, np.float64)
        olib().o64_write(self._h, _p(pos), _p(vel))

    def body_stats(self):
        out = np.zeros((self.nb, 13))
        olib().o64_body_stats(self._h, _p(out))
        return out

    def error(self):
        bits = C.c_uint32()
        body = C.c_int32()
        axis = np.zeros(3)
        olib().o64_error(self._h, C.byref(bits), C.byref(body), _p(axis))
        return bits.value, body.value, axis


def polar(a):
    a = np.ascontiguousarray(a, np.float64).reshape(9)
    r = np.zeros(9)
    q = np.zeros(4)
    ok = olib().oracle_polar(_p(a), _p(r), _p(q))
    return bool(ok), r.reshape(3, 3), q


def polar_warm(a, rq):
    a = np.ascontiguousarray(a, np.float64).reshape(9)
    rq = np.ascontiguousarray(rq, np.float32).reshape(4)
    r = np.zeros(9)
    q = np.zeros(4)
    ok = olib().oracle_polar_warm(_p(a), _p(rq), _p(r), _p(q))
    return bool(ok), r.reshape(3, 3), q


def sym_eigen(a):
    a = np.ascontiguousarray(a, np.float64).reshape(9)
    ev = np.zeros(3)
    vecs = np.zeros(9)
    olib().oracle_sym_eigen(_p(a), _p(ev), _p(vecs))
    return ev, vecs.reshape(3, 3)


def inertia_solve(I, dL):
    I = np.ascontiguousarray(I, np.float64).reshape(9)
    dL = np.ascontiguousarray(dL, np.float64)
    w = np.zeros(3)
    axis = np.zeros(3)
    st = olib().oracle_inertia_solve(_p(I), _p(dL), _p(w), _p(axis))
    return int(st), w, axis


def _f32(a, shape=None):
    a = np.ascontiguousarray(a, np.float32)
    return a if shape is None else a.reshape(shape)


def kat_ground(x, xinit, r, planes, relax=1.0):
    """planes: list of (point3, normal3, mu)."""
    pl = _f32([list(p) + list(n) + [mu] for p, n, mu in planes])
    out = np.zeros(3, np.float32)
    olib().oracle_kat_ground(_p(_f32(x)), _p(_f32(xinit)), r, len(planes), _p(pl), relax, _p(out))
    return out


def kat_pp(xi, wi, i, xj, wj, j, rr, relax=1.0):
    out = np.zeros(3, np.float32)
    olib().oracle_kat_pp(_p(_f32(xi)), wi, i, _p(_f32(xj)), wj, j, rr, relax, _p(out))
    return out


def kat_body_iteration(x, v, m, q0, dc, anchor, M, dt, init=None, incremental=True, linfix=True, angfix=True):
    x = _f32(x); n = len(x)
    init = x if init is None else _f32(init)
    xo = np.zeros((n, 3), np.float32)
    vo = np.zeros((n, 3), np.float32)
    err = olib().oracle_kat_body_iteration(n, _p(x), _p(_f32(v)), _p(_f32(m)), _p(_f32(q0)), _p(_f32(dc)),
                                           _p(init), _p(_f32(anchor)), M, dt, int(incremental), int(linfix),
                                           int(angfix), _p(xo), _p(vo))
    return int(err), xo, vo


def kat_momentum(m, xa, va, Pb, Lb, dt, linfix=True, angfix=True):
    xa = _f32(xa); n = len(xa)
    xo = np.zeros((n, 3), np.float32)
    vo = np.zeros((n, 3), np.float32)
    axis = np.zeros(3)
    err = olib().oracle_kat_momentum(n, _p(_f32(m)), _p(xa), _p(_f32(va)), _p(_f32(Pb)), _p(_f32(Lb)), dt,
                                     int(linfix), int(angfix), _p(xo), _p(vo), _p(axis))
    return int(err), xo, vo, axis


def _pack_mesh_call(fn, vertices, triangles, radius):
    v = np.ascontiguousarray(vertices, np.float64).reshape(-1, 3)
    t = np.ascontiguousarray(triangles, np.int32).reshape(-1, 3)
    cnt, cand, amb = C.c_long(), C.c_long(), C.c_long()
    cap = 1
    for _ in range(2):
        out = np.empty((cap, 3), np.float64)
        st = fn(_p(v), len(v), _p(t), len(t), radius, _p(out), cap, C.byref(cnt), C.byref(cand), C.byref(amb))
        if st != 0 or cnt.value <= cap:
            break
        cap = cnt.value
    return st, out[:cnt.value] if st == 0 else None, cand.value, amb.value


def pack_mesh(vertices, triangles, radius):
    """Oracle restatement of pack_mesh: (status, centers, candidates, ambiguous)."""
    return _pack_mesh_call(olib().oracle_pack_mesh, vertices, triangles, radius)


def ref_pack_mesh(vertices, triangles, radius):
    """The reference's own pack_mesh (oracle/_ref); None when not built."""
    L = rlib()
    return None if L is None else _pack_mesh_call(L.ref_pack_mesh, vertices, triangles, radius)

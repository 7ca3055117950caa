"""ctypes binding of the C-ABI in ``include/turbda_b200.h``.

This is the binding a maintainer of the reference would add on the Python
side and the path ``bench.py`` uses for device-resident
buffers (torch tensors, raw CUDA pointers).  It loads the in-tree
``paper_2407_12168_b200/lib/libturbda_b200.so`` and raises if it is missing:
there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libturbda_b200.so"

OK, CONFIG, DIMENSION, DIVERGED, DOMAIN, CUDA, INTERNAL, BLOWUP, ABORTED, SINGULAR, IO = range(11)
VARIANT_FREE_RUN, VARIANT_LETKF, VARIANT_ENSF = 0, 1, 2
SCORE_COMPONENTWISE, SCORE_JOINT = 0, 1
FP32, FP64 = 0, 1
INPUTS_ON_DEVICE = 0x1
ASYNC = 0x2
R_UNIFORM = 0x4
SHARDED = 0x8


class EnsfParams(C.Structure):
    _fields_ = [
        ("d_total", C.c_int64), ("k0", C.c_int64), ("d_local", C.c_int64),
        ("obs_dim", C.c_int64), ("n_members", C.c_int32), ("n_steps", C.c_int32),
        ("minibatch_j", C.c_int32), ("obs_kind", C.c_int32), ("eps", C.c_double),
        ("damping_t", C.c_double), ("relax_factor", C.c_double), ("seed", C.c_uint64),
        ("cycle", C.c_uint64), ("precision", C.c_int32), ("device", C.c_int32),
        ("device_count", C.c_int32), ("flags", C.c_uint32), ("score_mode", C.c_int32),
        ("reserved", C.c_int32),
    ]


class SqgParams(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("lx", C.c_double), ("ly", C.c_double),
                ("h", C.c_double), ("f", C.c_double), ("n", C.c_double), ("u0", C.c_double),
                ("hyper_order", C.c_int32), ("reserved", C.c_int32), ("hyper_efold", C.c_double),
                ("dt", C.c_double), ("drag_tau", C.c_double)]


class Experiment(C.Structure):
    _fields_ = [("sqg", SqgParams), ("variant", C.c_int32), ("model_quality", C.c_int32),
                ("cycles", C.c_int32), ("ensemble_size", C.c_int32),
                ("obs_interval", C.c_double), ("spinup_hours", C.c_double),
                ("clim_hours", C.c_double), ("seed", C.c_uint64), ("obs_r", C.c_double),
                ("obs_thinning", C.c_int32), ("obs_arctan", C.c_int32), ("n_steps", C.c_int32),
                ("minibatch_j", C.c_int32), ("eps", C.c_double), ("damping_t", C.c_double),
                ("relax_factor", C.c_double), ("precision", C.c_int32), ("score_mode", C.c_int32),
                ("me_enabled", C.c_int32), ("me_ncomp", C.c_int32),
                ("me_base_amplitude", C.c_double), ("me_prob", C.c_double * 8),
                ("me_frac", C.c_double * 8), ("letkf_cutoff_km", C.c_double),
                ("letkf_domain_km", C.c_double), ("letkf_rtps_alpha", C.c_double),
                ("letkf_obs_thinning", C.c_int32), ("reserved", C.c_int32)]


class LetkfParams(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("n_members", C.c_int32),
                ("obs_kind", C.c_int32), ("obs_dim", C.c_int64), ("cutoff_km", C.c_double),
                ("domain_km", C.c_double), ("rtps_alpha", C.c_double), ("device", C.c_int32),
                ("flags", C.c_uint32)]


class Status(C.Structure):
    _fields_ = [("code", C.c_int32), ("diverged_particle", C.c_int32),
                ("diverged_step", C.c_int32), ("reserved", C.c_int32),
                ("diverged_t", C.c_double), ("msg", C.c_char * 256)]


class TurbdaError(RuntimeError):
    def __init__(self, code: int, status: Status):
        self.code = code
        self.diverged_t = status.diverged_t
        self.diverged_particle = status.diverged_particle
        self.diverged_step = status.diverged_step
        super().__init__(f"turbda_b200 code {code}: {status.msg.decode(errors='replace')}")


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(make -C paper_2407_12168_b200/csrc)")
        L = C.CDLL(str(LIB_PATH))
        vp, dp = C.c_void_p, C.POINTER(C.c_double)
        L.turbda_ensf_params_init.argtypes = [C.POINTER(EnsfParams)]
        L.turbda_ensf_params_init.restype = None
        L.turbda_ensf_analyze.argtypes = [C.POINTER(EnsfParams), vp, vp, vp, vp, vp, vp,
                                          C.POINTER(Status)]
        L.turbda_ensf_analyze.restype = C.c_int
        L.turbda_ensf_analyze_rows.argtypes = [C.POINTER(EnsfParams), vp, vp, vp, vp, vp,
                                               C.POINTER(Status)]
        L.turbda_ensf_analyze_rows.restype = C.c_int
        L.turbda_ensf_check.argtypes = [C.c_int, C.POINTER(EnsfParams), C.POINTER(Status)]
        L.turbda_ensf_check.restype = C.c_int
        L.turbda_relax_spread.argtypes = [vp, vp, C.c_int32, C.c_int64, C.c_double, vp,
                                          C.c_int32, C.c_uint32, vp, C.POINTER(Status)]
        L.turbda_relax_spread.restype = C.c_int
        L.turbda_score.argtypes = [vp, C.c_int64, C.c_double, vp, C.c_int32, vp, C.c_int32,
                                   C.c_double, vp, vp, vp, C.c_int64, C.c_int32, C.c_double, vp,
                                   C.c_int32, C.POINTER(Status)]
        L.turbda_score.restype = C.c_int
        L.turbda_diag.argtypes = [vp, C.c_int32, C.c_int64, vp, dp, C.c_int32, C.c_uint32, vp,
                                  C.POINTER(Status)]
        L.turbda_diag.restype = C.c_int
        L.turbda_device_count.restype = C.c_int
        L.turbda_abi_version.restype = C.c_int
        L.turbda_build_arch.restype = C.c_char_p
        L.turbda_launch_count.restype = C.c_uint64
        L.turbda_profile_enable.argtypes = [C.c_int]
        L.turbda_profile_enable.restype = None
        L.turbda_profile_read.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_uint64)]
        L.turbda_profile_read.restype = C.c_int
        L.turbda_comm_unique_id.argtypes = [C.c_void_p, C.POINTER(Status)]
        L.turbda_comm_unique_id.restype = C.c_int
        L.turbda_comm_init.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.POINTER(Status)]
        L.turbda_comm_init.restype = C.c_int
        L.turbda_comm_destroy.argtypes = [C.c_int32]
        L.turbda_comm_destroy.restype = C.c_int
        L.turbda_sqg_params_init.argtypes = [C.POINTER(SqgParams)]
        L.turbda_sqg_params_init.restype = None
        L.turbda_sqg_create.argtypes = [C.POINTER(SqgParams), C.c_int32, C.c_int32,
                                        C.POINTER(C.c_void_p), C.POINTER(Status)]
        L.turbda_sqg_create.restype = C.c_int
        L.turbda_sqg_advance.argtypes = [C.c_void_p, vp, C.c_double, C.c_uint32, vp, dp,
                                         C.POINTER(Status)]
        L.turbda_sqg_advance.restype = C.c_int
        L.turbda_sqg_destroy.argtypes = [C.c_void_p]
        L.turbda_sqg_destroy.restype = C.c_int
        L.turbda_nature_run.argtypes = [C.POINTER(SqgParams), C.c_double, C.c_double, C.c_double,
                                        C.c_uint64, vp, C.c_int32, C.POINTER(C.c_int32),
                                        C.c_int32, C.POINTER(Status)]
        L.turbda_nature_run.restype = C.c_int
        L.turbda_experiment_init.argtypes = [C.POINTER(Experiment)]
        L.turbda_experiment_init.restype = None
        L.turbda_run_experiment.argtypes = [C.POINTER(Experiment), C.c_int32, vp, C.c_int32,
                                            C.POINTER(C.c_int32), dp, vp, C.POINTER(Status)]
        L.turbda_run_experiment.restype = C.c_int
        L.turbda_letkf_params_init.argtypes = [C.POINTER(LetkfParams)]
        L.turbda_letkf_params_init.restype = None
        L.turbda_letkf_analyze.argtypes = [C.POINTER(LetkfParams), vp, vp, vp, vp, vp, vp, vp,
                                           C.POINTER(Status)]
        L.turbda_letkf_analyze.restype = C.c_int
        L.turbda_rtps_inflate.argtypes = [vp, vp, C.c_int32, C.c_int64, C.c_double, vp,
                                          C.c_int32, C.c_uint32, vp, C.POINTER(Status)]
        L.turbda_rtps_inflate.restype = C.c_int
        L.turbda_gaspari_cohn.argtypes = [C.c_double, dp, C.POINTER(Status)]
        L.turbda_gaspari_cohn.restype = C.c_int
        L.turbda_snapshot_write.argtypes = [C.c_char_p, vp, C.c_int32, C.c_int32, C.c_int32,
                                            C.c_double, C.c_uint32, C.POINTER(Status)]
        L.turbda_snapshot_write.restype = C.c_int
        L.turbda_snapshot_read.argtypes = [C.c_char_p, vp, C.c_int32, C.POINTER(C.c_int32),
                                           C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                           C.POINTER(C.c_double), C.c_uint32, C.POINTER(Status)]
        L.turbda_snapshot_read.restype = C.c_int
        _lib = L
    return _lib


def params(**kw) -> EnsfParams:
    p = EnsfParams()
    lib().turbda_ensf_params_init(C.byref(p))
    for k, v in kw.items():
        if not hasattr(p, k):
            raise TypeError(f"unknown turbda_ensf_params field {k!r}")
        setattr(p, k, v)
    return p


def _check(code: int, st: Status):
    if code != OK:
        raise TurbdaError(code, st)


def _ptr(a) -> int | None:
    """numpy array -> host address; torch tensor / int -> address; None -> NULL."""
    if a is None:
        return None
    if isinstance(a, int):
        return a
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    raise TypeError(type(a))


def analyze(p: EnsfParams, forecast, y, r_diag, obs_idx, out, stream: int | None = None):
    """Raw C-ABI call.  With ``p.flags & INPUTS_ON_DEVICE`` every array is a
    device buffer (torch CUDA tensor or int address) and ``stream`` a
    cudaStream_t handle; otherwise numpy host arrays."""
    st = Status()
    code = lib().turbda_ensf_analyze(C.byref(p), _ptr(forecast), _ptr(y), _ptr(r_diag),
                                     _ptr(obs_idx), _ptr(out), stream, C.byref(st))
    _check(code, st)
    return st


def analyze_rows(p: EnsfParams, forecast_rows, y, r_diag, obs_idx, analysis_rows):
    """Raw C-ABI call with one host pointer per member row in and out (the
    reference ``Ensemble::members`` layout): ``forecast_rows`` /
    ``analysis_rows`` are ctypes ``c_void_p`` arrays of length n_members."""
    st = Status()
    code = lib().turbda_ensf_analyze_rows(C.byref(p), C.cast(forecast_rows, C.c_void_p), _ptr(y),
                                          _ptr(r_diag), _ptr(obs_idx),
                                          C.cast(analysis_rows, C.c_void_p), C.byref(st))
    _check(code, st)
    return st


def check(device: int, p: EnsfParams) -> Status:
    st = Status()
    _check(lib().turbda_ensf_check(device, C.byref(p), C.byref(st)), st)
    return st


def analyze_host(members, y, r=1.0, idx=None, *, n_steps=100, eps=0.01, minibatch_j=0,
                 damping_t=1.0, relax_factor=1.0, seed=7, cycle=1, precision=FP32, device=-1,
                 device_count=1, k0=0, d_total=None, arctan=False, joint=False,
                 r_uniform=False, sharded=False):
    """numpy-in / numpy-out analysis over the window [k0, k0 + d) of a state
    of dimension d_total (defaults to the whole state).  ``r_uniform``: pass
    the scalar ``r`` once (TURBDA_R_UNIFORM) instead of an obs_dim copy.
    ``sharded``: this rank's window of a state split over the device's
    communicator (TURBDA_SHARDED; every rank makes the same call)."""
    x = np.ascontiguousarray(members, dtype=np.float64)
    m, d = x.shape
    y = np.ascontiguousarray(y, dtype=np.float64)
    if r_uniform:
        r = np.array([float(r)], np.float64)
    else:
        r = np.ascontiguousarray(np.broadcast_to(np.asarray(r, np.float64), y.shape))
    ix = None if idx is None else np.ascontiguousarray(idx, dtype=np.int64)
    p = params(d_total=d if d_total is None else d_total, k0=k0, d_local=d, obs_dim=y.size,
               n_members=m, n_steps=n_steps, minibatch_j=minibatch_j,
               obs_kind=(0 if idx is None else 1) + (2 if arctan else 0), eps=eps,
               damping_t=damping_t,
               relax_factor=relax_factor, seed=seed, cycle=cycle, precision=precision,
               device=device, device_count=device_count,
               score_mode=SCORE_JOINT if joint else SCORE_COMPONENTWISE,
               flags=(R_UNIFORM if r_uniform else 0) | (SHARDED if sharded else 0))
    out = np.empty_like(x)
    analyze(p, x, y, r, ix, out)
    return out


def letkf_params(**kw) -> LetkfParams:
    p = LetkfParams()
    lib().turbda_letkf_params_init(C.byref(p))
    for k, v in kw.items():
        if not hasattr(p, k):
            raise TypeError(f"unknown turbda_letkf_params field {k!r}")
        setattr(p, k, v)
    return p


def letkf_raw(p: LetkfParams, forecast, y, r_diag, obs_idx, locations, out,
              stream: int | None = None):
    """Raw C-ABI call (host numpy arrays, or device buffers with
    ``p.flags & INPUTS_ON_DEVICE``)."""
    st = Status()
    code = lib().turbda_letkf_analyze(C.byref(p), _ptr(forecast), _ptr(y), _ptr(r_diag),
                                      _ptr(obs_idx), _ptr(locations), _ptr(out), stream,
                                      C.byref(st))
    _check(code, st)


def letkf_analyze(members, y, r=1.0, idx=None, *, nx, ny, cutoff_km=2000.0, domain_km=20000.0,
                  rtps_alpha=0.3, arctan=False, locations=None, device=-1, r_uniform=False):
    """numpy-in / numpy-out LETKF analysis of an (M, 2*nx*ny) ensemble."""
    x = np.ascontiguousarray(members, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    if r_uniform:
        rr = np.array([float(r)], np.float64)
    else:
        rr = np.ascontiguousarray(np.broadcast_to(np.asarray(r, np.float64), y.shape))
    ix = None if idx is None else np.ascontiguousarray(idx, dtype=np.int64)
    loc = None if locations is None else np.ascontiguousarray(locations, dtype=np.float64)
    p = letkf_params(nx=nx, ny=ny, n_members=x.shape[0],
                     obs_kind=(0 if idx is None else 1) + (2 if arctan else 0), obs_dim=y.size,
                     cutoff_km=cutoff_km, domain_km=domain_km, rtps_alpha=rtps_alpha,
                     device=device, flags=R_UNIFORM if r_uniform else 0)
    if x.shape[1] != 2 * nx * ny:
        raise TurbdaError(DIMENSION, _status_msg("letkf_analyze: state/grid size mismatch"))
    out = np.empty_like(x)
    letkf_raw(p, x, y, rr, ix, loc, out)
    return out


def rtps_inflate(analysis, background, alpha, device=-1):
    a = np.ascontiguousarray(analysis, np.float64)
    b = np.ascontiguousarray(background, np.float64)
    out = np.empty_like(a)
    st = Status()
    _check(lib().turbda_rtps_inflate(_ptr(a), _ptr(b), a.shape[0], a.shape[1], alpha, _ptr(out),
                                     device, 0, None, C.byref(st)), st)
    return out


def gaspari_cohn(r: float) -> float:
    v = C.c_double()
    st = Status()
    _check(lib().turbda_gaspari_cohn(r, C.byref(v), C.byref(st)), st)
    return v.value


def snapshot_write(path, states, time_hours=0.0, flags=0):
    """SQGSNAP v1: `states` (..., 2, ny, nx) float64 (numpy, or a CUDA tensor
    with flags=INPUTS_ON_DEVICE), one snapshot per leading index."""
    shape = tuple(states.shape)
    ny, nx = shape[-2], shape[-1]
    count = int(np.prod(shape[:-3])) if len(shape) > 3 else 1
    a = states if flags & INPUTS_ON_DEVICE else np.ascontiguousarray(states, np.float64)
    st = Status()
    _check(lib().turbda_snapshot_write(str(path).encode(), _ptr(a), count, nx, ny, time_hours,
                                       flags, C.byref(st)), st)


def snapshot_read(path, max_count=1 << 20):
    """-> (states [count, 2, ny, nx], time_hours)"""
    n, nx, ny, t = C.c_int32(), C.c_int32(), C.c_int32(), C.c_double()
    st = Status()
    _check(lib().turbda_snapshot_read(str(path).encode(), None, max_count, C.byref(n), C.byref(nx),
                                      C.byref(ny), C.byref(t), 0, C.byref(st)), st)
    out = np.empty((n.value, 2, ny.value, nx.value), np.float64)
    _check(lib().turbda_snapshot_read(str(path).encode(), _ptr(out), n.value, C.byref(n),
                                      C.byref(nx), C.byref(ny), C.byref(t), 0, C.byref(st)), st)
    return out, t.value


def _status_msg(msg: str) -> Status:
    st = Status()
    st.msg = msg.encode()[:255]
    return st


def score(z, t, members, batch=None, eps=0.01, y=None, r=None, idx=None, damping_t=1.0,
          device=-1, arctan=False):
    z = np.ascontiguousarray(z, np.float64)
    x = np.ascontiguousarray(members, np.float64)
    b = None if batch is None else np.ascontiguousarray(batch, np.int32)
    out = np.empty_like(z)
    yy = rr = ii = None
    nobs = 0
    if y is not None:
        yy = np.ascontiguousarray(y, np.float64)
        rr = np.ascontiguousarray(np.broadcast_to(np.asarray(r, np.float64), yy.shape))
        ii = None if idx is None else np.ascontiguousarray(idx, np.int64)
        nobs = yy.size
    st = Status()
    code = lib().turbda_score(_ptr(z), z.size, t, _ptr(x), x.shape[0], _ptr(b),
                              0 if b is None else b.size, eps, _ptr(yy), _ptr(rr), _ptr(ii),
                              nobs, (0 if idx is None else 1) + (2 if arctan else 0), damping_t,
                              _ptr(out), device,
                              C.byref(st))
    _check(code, st)
    return out


def relax_spread(analysis, forecast, factor, device=-1):
    a = np.ascontiguousarray(analysis, np.float64)
    f = np.ascontiguousarray(forecast, np.float64)
    out = np.empty_like(a)
    st = Status()
    _check(lib().turbda_relax_spread(_ptr(a), _ptr(f), a.shape[0], a.shape[1], factor,
                                     _ptr(out), device, 0, None, C.byref(st)), st)
    return out


def diag(members, truth=None, device=-1, sharded=False):
    """(sum (mean - truth)^2, sum dev^2) in a fixed order; ``sharded``: the
    arrays are this rank's shard and the sums are allreduced over the
    device's communicator (TURBDA_SHARDED)."""
    x = np.ascontiguousarray(members, np.float64)
    t = None if truth is None else np.ascontiguousarray(truth, np.float64)
    out = (C.c_double * 2)()
    st = Status()
    _check(lib().turbda_diag(_ptr(x), x.shape[0], x.shape[1], _ptr(t), out, device,
                             SHARDED if sharded else 0, None, C.byref(st)), st)
    return float(out[0]), float(out[1])


def comm_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    st = Status()
    _check(lib().turbda_comm_unique_id(buf, C.byref(st)), st)
    return bytes(buf)


def comm_init(device: int, rank: int, world: int, uid: bytes) -> None:
    """Library NCCL communicator for a state sharded over `world` processes
    (used by the joint score mode's per-step allreduce)."""
    buf = (C.c_char * 128).from_buffer_copy(uid)
    st = Status()
    _check(lib().turbda_comm_init(device, rank, world, buf, C.byref(st)), st)


def comm_destroy(device: int) -> None:
    lib().turbda_comm_destroy(device)


def sqg_params(**kw) -> SqgParams:
    p = SqgParams()
    lib().turbda_sqg_params_init(C.byref(p))
    for k, v in kw.items():
        setattr(p, k, v)
    return p


class SqgModel:
    """Batched GPU SQG stepper (turbda_sqg_*): advance(states, hours) on an
    (batch, 2, ny, nx) float64 numpy array, in place."""

    def __init__(self, batch=1, device=-1, **params):
        self.p = sqg_params(**params)
        self.batch = batch
        self.h = C.c_void_p()
        st = Status()
        _check(lib().turbda_sqg_create(C.byref(self.p), batch, device, C.byref(self.h),
                                       C.byref(st)), st)
        self.max_cfl = 0.0

    def advance(self, states, hours):
        a = np.ascontiguousarray(states, np.float64)
        cfl = C.c_double(self.max_cfl)
        st = Status()
        _check(lib().turbda_sqg_advance(self.h, a.ctypes.data, hours, 0, None, C.byref(cfl),
                                        C.byref(st)), st)
        self.max_cfl = cfl.value
        return a

    def __del__(self):
        if getattr(self, "h", None) and self.h.value:
            lib().turbda_sqg_destroy(self.h)
            self.h = C.c_void_p()


def nature_run(spinup, duration, interval, seed, device=-1, **params):
    p = sqg_params(**params)
    n = int(round(duration / interval)) + 1
    out = np.empty((n, 2 * p.nx * p.ny), np.float64)
    got = C.c_int32(0)
    st = Status()
    _check(lib().turbda_nature_run(C.byref(p), spinup, duration, interval, seed,
                                   out.ctypes.data, n, C.byref(got), device, C.byref(st)), st)
    return out[: got.value]


def experiment(**kw) -> Experiment:
    e = Experiment()
    lib().turbda_experiment_init(C.byref(e))
    for k, v in kw.items():
        setattr(e, k, v)
    return e


def run_experiment_raw(e: Experiment, device=-1, phases=None):
    """(records [n][6], max_cfl); raises TurbdaError (records of completed
    cycles in err.partial on TURBDA_ABORTED).  ``phases``: optional float64[4]
    receiving the device seconds of nature run / forecasts / analyses / diagnostics."""
    rec = np.zeros((max(e.cycles, 1), 6), np.float64)
    n = C.c_int32(0)
    cfl = C.c_double(0)
    st = Status()
    code = lib().turbda_run_experiment(C.byref(e), device, rec.ctypes.data, e.cycles,
                                       C.byref(n), C.byref(cfl),
                                       None if phases is None else phases.ctypes.data,
                                       C.byref(st))
    if code != OK:
        err = TurbdaError(code, st)
        err.partial = rec[: n.value]
        raise err
    return rec[: n.value], cfl.value


class Probe(C.Structure):
    _fields_ = [("n_cycles", C.c_int32), ("cycles", C.c_void_p), ("k0", C.c_int64),
                ("width", C.c_int64), ("forecast", C.c_void_p), ("analysis", C.c_void_p),
                ("y", C.c_void_p)]


def run_experiment_probe(e: Experiment, cycles, k0: int, width: int, obs_dim: int, device=-1):
    """The experiment plus an open-loop probe (turbda_run_experiment_probe):
    returns (records, {cycle: (forecast [m][width], analysis [m][width],
    y [obs_dim])}) for the listed cycles."""
    L = lib()
    if not hasattr(L, "_probe_bound"):
        L.turbda_run_experiment_probe.argtypes = [C.POINTER(Experiment), C.c_int32, C.c_void_p,
                                                  C.c_int32, C.POINTER(C.c_int32),
                                                  C.POINTER(C.c_double), C.c_void_p,
                                                  C.POINTER(Probe), C.POINTER(Status)]
        L.turbda_run_experiment_probe.restype = C.c_int
        L._probe_bound = True
    cyc = np.ascontiguousarray(sorted(cycles), np.int32)
    m = e.ensemble_size
    fc = np.zeros((cyc.size, m, width))
    an = np.zeros((cyc.size, m, width))
    yy = np.zeros((cyc.size, obs_dim))
    pr = Probe(int(cyc.size), cyc.ctypes.data, int(k0), int(width), fc.ctypes.data,
               an.ctypes.data, yy.ctypes.data)
    rec = np.zeros((max(e.cycles, 1), 6), np.float64)
    n = C.c_int32(0)
    cfl = C.c_double(0)
    st = Status()
    _check(L.turbda_run_experiment_probe(C.byref(e), device, rec.ctypes.data, e.cycles,
                                         C.byref(n), C.byref(cfl), None, C.byref(pr),
                                         C.byref(st)), st)
    return rec[: n.value], {int(c): (fc[q], an[q], yy[q]) for q, c in enumerate(cyc)}


def device_count() -> int:
    return int(lib().turbda_device_count())


def launch_count() -> int:
    return int(lib().turbda_launch_count())


def profile_enable(on: bool = True) -> None:
    lib().turbda_profile_enable(1 if on else 0)


def profile_read() -> tuple[float, int]:
    """(summed fused-kernel ms, timed launches) since the previous read."""
    ms, n = C.c_double(), C.c_uint64()
    lib().turbda_profile_read(C.byref(ms), C.byref(n))
    return float(ms.value), int(n.value)


def exported_symbols() -> list[str]:
    """Symbols include/turbda_b200.h declares (checked by the CPU tests)."""
    hdr = Path(__file__).resolve().parents[1] / "include" / "turbda_b200.h"
    import re
    return sorted(set(re.findall(r"\b(turbda_[a-z0-9_]+)\s*\(", hdr.read_text())))


if os.environ.get("TURBDA_B200_EAGER_LOAD"):
    lib()

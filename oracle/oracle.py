"""TEST INFRASTRUCTURE ONLY - ctypes access to the two CPU oracles.

* ``RefOracle``  -- the *unmodified* reference hot path
  (``/root/reference/proj/src/{ensf,ensemble,observation,rng,parallel}.cpp``)
  compiled by ``oracle/Makefile`` into ``oracle/_ref/*/libturbda_ref.so``
  behind ``oracle/ref_shim.cpp``.  ``kind == "reference"``.
* ``PortOracle`` -- the plain-C restatement ``oracle/ensf_oracle.c``
  (``oracle/_build/libensf_oracle.so``).  ``kind == "port"``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this module; the
product package never does.  Neither library needs ``/root/reference`` at
run time: both are prebuilt and travel with the gpurun snapshot.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
STATUS = {0: "ok", 1: "config", 2: "dimension", 3: "diverged", 4: "domain", 5: "other"}

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip64 = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_ip32 = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_up32 = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
_up64 = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str = "", diverged_t: float | None = None):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.kind = STATUS.get(code, str(code))
        self.diverged_t = diverged_t


def _cpu_flags() -> set[str]:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("flags"):
                    return set(line.split(":", 1)[1].split())
    except OSError:
        pass
    return set()


def _ref_lib_path() -> Path:
    """Pick the -march=native build when this CPU has every ISA flag of the
    build host, otherwise the x86-64-v3 build."""
    native = HERE / "_ref" / "native" / "libturbda_ref.so"
    portable = HERE / "_ref" / "portable" / "libturbda_ref.so"
    flags_file = HERE / "_ref" / "build_cpu_flags.txt"
    if native.exists() and flags_file.exists():
        if set(flags_file.read_text().split()) <= _cpu_flags():
            return native
    return portable


def ref_available() -> bool:
    return _ref_lib_path().exists()


def port_available() -> bool:
    return (HERE / "_build" / "libensf_oracle.so").exists()


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def _obs_arrays(d, y, r, idx, arctan=False):
    y = np.ascontiguousarray(y, dtype=np.float64)
    r = np.broadcast_to(np.asarray(r, dtype=np.float64), y.shape).copy()
    if idx is None:
        return y, r, np.zeros(1, np.int64), 2 if arctan else 0
    return y, r, np.ascontiguousarray(idx, dtype=np.int64), 3 if arctan else 1


class RefOracle:
    kind = "reference"

    def __init__(self, path: str | os.PathLike | None = None):
        self.path = Path(path) if path else _ref_lib_path()
        L = self.lib = C.CDLL(str(self.path))
        L.ref_analyze.restype = C.c_int
        L.ref_analyze.argtypes = [_dp, C.c_int, C.c_int64, _dp, _dp, _ip64, C.c_int64, C.c_int,
                                  C.c_int, C.c_double, C.c_int, C.c_double, C.c_double,
                                  C.c_uint64, C.c_uint64, C.c_int, _dp,
                                  C.POINTER(C.c_double), C.c_char_p, C.c_int]
        L.ref_relax_spread.restype = C.c_int
        L.ref_relax_spread.argtypes = [_dp, _dp, C.c_int, C.c_int64, C.c_double, _dp]
        L.ref_prior_score.restype = C.c_int
        L.ref_prior_score.argtypes = [_dp, C.c_int64, C.c_double, _dp, C.c_int, _ip32, C.c_int,
                                      C.c_double, _dp]
        L.ref_posterior_score.restype = C.c_int
        L.ref_posterior_score.argtypes = [_dp, C.c_int64, C.c_double, _dp, C.c_int, _dp, _dp,
                                          _ip64, C.c_int64, C.c_int, C.c_double, C.c_double, _dp]
        L.ref_philox4x32.restype = None
        L.ref_philox4x32.argtypes = [_up32, _up32, _up32]
        L.ref_splitmix64.restype = C.c_uint64
        L.ref_splitmix64.argtypes = [C.c_uint64]
        for name in ("ref_stream_normals", "ref_stream_uniforms"):
            getattr(L, name).restype = None
            getattr(L, name).argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_int64, _dp]
        L.ref_stream_u64.restype = None
        L.ref_stream_u64.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_int64, _up64]
        L.ref_fast_exp_nonpos.restype = C.c_double
        L.ref_fast_exp_nonpos.argtypes = [C.c_double]
        L.ref_synthesize_obs.restype = C.c_int
        L.ref_synthesize_obs.argtypes = [_dp, C.c_int64, _ip64, C.c_int64, C.c_int, C.c_double,
                                         C.c_uint64, C.c_uint64, _dp]
        L.ref_rmse.restype = C.c_double
        L.ref_rmse.argtypes = [_dp, _dp, C.c_int64]
        L.ref_spread.restype = C.c_double
        L.ref_spread.argtypes = [_dp, C.c_int, C.c_int64]

    # -- analysis ---------------------------------------------------------
    def analyze(self, members, y, r=1.0, idx=None, *, n_steps=100, eps=0.01, minibatch_j=0,
                damping_t=1.0, relax_factor=1.0, seed=7, cycle=1, workers=0):
        x = np.ascontiguousarray(members, dtype=np.float64)
        m, d = x.shape
        y, r, idx_a, kind = _obs_arrays(d, y, r, idx)
        out = np.empty_like(x)
        div_t = C.c_double(float("nan"))
        msg = C.create_string_buffer(256)
        code = self.lib.ref_analyze(x, m, d, y, r, idx_a, y.size, kind, n_steps, eps,
                                    minibatch_j, damping_t, relax_factor, seed, cycle,
                                    workers, out, C.byref(div_t), msg, 256)
        if code:
            raise OracleError(code, msg.value.decode(), div_t.value)
        return out

    def relax_spread(self, analysis, forecast, factor):
        a = np.ascontiguousarray(analysis, dtype=np.float64)
        f = np.ascontiguousarray(forecast, dtype=np.float64)
        out = np.empty_like(a)
        code = self.lib.ref_relax_spread(a, f, a.shape[0], a.shape[1], factor, out)
        if code:
            raise OracleError(code)
        return out

    def prior_score(self, z, t, members, batch=(), eps=0.01):
        z = np.ascontiguousarray(z, dtype=np.float64)
        x = np.ascontiguousarray(members, dtype=np.float64)
        b = np.ascontiguousarray(batch, dtype=np.int32) if len(batch) else np.zeros(1, np.int32)
        out = np.empty_like(z)
        code = self.lib.ref_prior_score(z, z.size, t, x, x.shape[0], b, len(batch), eps, out)
        if code:
            raise OracleError(code)
        return out

    def posterior_score(self, z, t, members, y, r=1.0, idx=None, eps=0.01, damping_t=1.0):
        z = np.ascontiguousarray(z, dtype=np.float64)
        x = np.ascontiguousarray(members, dtype=np.float64)
        y, r, idx_a, kind = _obs_arrays(z.size, y, r, idx)
        out = np.empty_like(z)
        code = self.lib.ref_posterior_score(z, z.size, t, x, x.shape[0], y, r, idx_a, y.size,
                                            kind, eps, damping_t, out)
        if code:
            raise OracleError(code)
        return out

    # -- rng / utilities ---------------------------------------------------
    def philox4x32(self, ctr, key):
        out = np.zeros(4, np.uint32)
        self.lib.ref_philox4x32(np.asarray(ctr, np.uint32), np.asarray(key, np.uint32), out)
        return out

    def splitmix64(self, x):
        return int(self.lib.ref_splitmix64(x))

    def stream_normals(self, seed, use, entity, n):
        out = np.empty(n, np.float64)
        self.lib.ref_stream_normals(seed, use, entity, n, out)
        return out

    def stream_uniforms(self, seed, use, entity, n):
        out = np.empty(n, np.float64)
        self.lib.ref_stream_uniforms(seed, use, entity, n, out)
        return out

    def stream_u64(self, seed, use, entity, n):
        out = np.empty(n, np.uint64)
        self.lib.ref_stream_u64(seed, use, entity, n, out)
        return out

    def fast_exp_nonpos(self, x):
        return float(self.lib.ref_fast_exp_nonpos(x))

    def synthesize_obs(self, truth, r_variance, seed, cycle, idx=None):
        t = np.ascontiguousarray(truth, dtype=np.float64)
        idx_a = np.zeros(1, np.int64) if idx is None else np.ascontiguousarray(idx, np.int64)
        n = t.size if idx is None else idx_a.size
        out = np.empty(n, np.float64)
        code = self.lib.ref_synthesize_obs(t, t.size, idx_a, n, 0 if idx is None else 1,
                                           r_variance, seed, cycle, out)
        if code:
            raise OracleError(code)
        return out

    def rmse(self, mean, truth):
        return float(self.lib.ref_rmse(np.ascontiguousarray(mean, np.float64),
                                       np.ascontiguousarray(truth, np.float64), len(mean)))

    def spread(self, members):
        x = np.ascontiguousarray(members, np.float64)
        return float(self.lib.ref_spread(x, x.shape[0], x.shape[1]))


class PortOracle:
    kind = "port"

    def __init__(self, path: str | os.PathLike | None = None):
        self.path = Path(path) if path else HERE / "_build" / "libensf_oracle.so"
        L = self.lib = C.CDLL(str(self.path))
        L.orc_analyze.restype = C.c_int
        L.orc_analyze.argtypes = [_dp, C.c_int, C.c_int64, C.c_int64, C.c_int64, _dp, _dp, _ip64,
                                  C.c_int64, C.c_int, C.c_int, C.c_double, C.c_int, C.c_double,
                                  C.c_double, C.c_uint64, C.c_uint64, C.c_int, _dp,
                                  C.POINTER(C.c_double), C.c_int]
        L.orc_philox4x32.restype = None
        L.orc_philox4x32.argtypes = [_up32, _up32, _up32]
        L.orc_splitmix64.restype = C.c_uint64
        L.orc_splitmix64.argtypes = [C.c_uint64]
        L.orc_stream_key.restype = C.c_uint64
        L.orc_stream_key.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_stream_normal.restype = C.c_double
        L.orc_stream_normal.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.orc_stream_u64.restype = C.c_uint64
        L.orc_stream_u64.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.orc_stream_normals.restype = None
        L.orc_stream_normals.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_int64,
                                         C.c_int64, _dp]
        L.orc_fast_exp_nonpos.restype = C.c_double
        L.orc_fast_exp_nonpos.argtypes = [C.c_double]
        L.orc_batch_table.restype = None
        L.orc_batch_table.argtypes = [C.c_uint64, C.c_uint64, C.c_int, C.c_int, C.c_int, _ip32]
        L.orc_relax_spread.restype = C.c_int
        L.orc_relax_spread.argtypes = [_dp, _dp, C.c_int, C.c_int64, C.c_double, _dp]

    def analyze(self, members, y, r=1.0, idx=None, *, n_steps=100, eps=0.01, minibatch_j=0,
                damping_t=1.0, relax_factor=1.0, seed=7, cycle=1, workers=0, k0=0,
                d_total=None, arctan=False, joint=False):
        """``members`` is the [m][dl] window starting at global coordinate k0.
        ``arctan=True``: h(x) = atan(x); ``joint=True``: joint-norm weights
        (both extensions, parity unpinned)."""
        x = np.ascontiguousarray(members, dtype=np.float64)
        m, dl = x.shape
        d_total = dl if d_total is None else d_total
        y, r, idx_a, kind = _obs_arrays(dl, y, r, idx, arctan)
        out = np.empty_like(x)
        div_t = C.c_double(float("nan"))
        workers = workers if workers > 0 else host_cores()
        code = self.lib.orc_analyze(x, m, dl, k0, d_total, y, r, idx_a, y.size, kind, n_steps,
                                    eps, minibatch_j, damping_t, relax_factor, seed, cycle,
                                    workers, out, C.byref(div_t), 1 if joint else 0)
        if code:
            raise OracleError(code, "", div_t.value)
        return out

    def philox4x32(self, ctr, key):
        out = np.zeros(4, np.uint32)
        self.lib.orc_philox4x32(np.asarray(ctr, np.uint32), np.asarray(key, np.uint32), out)
        return out

    def splitmix64(self, x):
        return int(self.lib.orc_splitmix64(x))

    def stream_normals(self, seed, use, entity, n, n0=0):
        out = np.empty(n, np.float64)
        self.lib.orc_stream_normals(seed, use, entity, n0, n, out)
        return out

    def stream_u64(self, seed, use, entity, n):
        key = self.lib.orc_stream_key(seed, use)
        return np.array([self.lib.orc_stream_u64(key, entity, q) for q in range(n)], np.uint64)

    def fast_exp_nonpos(self, x):
        return float(self.lib.orc_fast_exp_nonpos(x))

    def batch_table(self, seed, cycle, m, j_batch, n_steps):
        out = np.empty(n_steps * j_batch, np.int32)
        self.lib.orc_batch_table(seed, cycle, m, j_batch, n_steps, out)
        return out.reshape(n_steps, j_batch)

    def relax_spread(self, analysis, forecast, factor):
        a = np.ascontiguousarray(analysis, dtype=np.float64)
        f = np.ascontiguousarray(forecast, dtype=np.float64)
        out = np.empty_like(a)
        self.lib.orc_relax_spread(a, f, a.shape[0], a.shape[1], factor, out)
        return out


def rel_l2(a, b) -> float:
    """Relative L2 error, proj/tests/helpers.hpp:65-72 (``rel_err``).

    Non-finite entries must coincide exactly (same inf sign / nan position);
    they then drop out of the norm.  A mismatch there returns inf."""
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    if a.shape != b.shape:
        return float("inf")
    fa, fb = np.isfinite(a), np.isfinite(b)
    if not np.array_equal(fa, fb):
        return float("inf")
    if not fa.all():
        na, nb = a[~fa], b[~fb]
        if not np.array_equal(np.isnan(na), np.isnan(nb)) or \
                not np.array_equal(na[~np.isnan(na)], nb[~np.isnan(nb)]):
            return float("inf")
        a, b = a[fa], b[fb]
    den = np.sum(b * b)
    num = np.sum((a - b) ** 2)
    if den == 0.0:
        return 0.0 if num == 0.0 else float("inf")
    return float(np.sqrt(num / den))


# -- synthetic inputs, SURVEY.md section 8(d) -------------------------------
STREAM_GENERIC = 8
STREAM_OBS_NOISE = 5


def throughput_inputs(m, d, oracle=None, stride=0):
    """x_jk = RngStream(1234, generic, j).normal(); y = RngStream(99, obs_noise, 1).normal()."""
    o = oracle or PortOracle()
    x = np.stack([o.stream_normals(1234, STREAM_GENERIC, j, d) for j in range(m)])
    nobs = d if stride <= 1 else len(range(0, d, stride))
    y = o.stream_normals(99, STREAM_OBS_NOISE, 1, nobs)
    idx = None if stride <= 1 else np.arange(0, d, stride, dtype=np.int64)
    return x, y, idx


def conditioned_inputs(m, d, oracle=None, stride=0):
    """truth_k = 2 sin(0.001 k) + 0.5 N; x_jk = truth_k + N; y = H(truth) + N."""
    o = oracle or PortOracle()
    k = np.arange(d, dtype=np.float64)
    truth = 2.0 * np.sin(0.001 * k) + 0.5 * o.stream_normals(5, STREAM_GENERIC, 77, d)
    x = np.stack([truth + o.stream_normals(1234, STREAM_GENERIC, j, d) for j in range(m)])
    idx = None if stride <= 1 else np.arange(0, d, stride, dtype=np.int64)
    ht = truth if idx is None else truth[idx]
    y = ht + o.stream_normals(99, STREAM_OBS_NOISE, 1, ht.size)
    return x, y, idx, truth


class RefCycleOracle:
    """The reference's cycle driver, SQG model and LETKF (proj/src/{osse,
    config,forecast,sqg,spectral,letkf}.cpp + the hot path), unmodified,
    built against cuFFTW and the Eigen subset in oracle/ref_shadow/Eigen
    (oracle/ref_cycle_shim.cpp).  Needs a GPU at run time for the model
    (cuFFTW); ``letkf_analyze`` is CPU only."""

    kind = "reference"

    def __init__(self, path=None):
        self.path = Path(path) if path else HERE / "_ref" / "libturbda_ref_cycle.so"
        L = self.lib = C.CDLL(str(self.path))
        L.refc_run_experiment.restype = C.c_int
        L.refc_run_experiment.argtypes = [C.c_char_p, C.c_int, _dp, C.c_int,
                                          C.POINTER(C.c_int), C.c_char_p, C.c_int]
        L.refc_sqg_advance.restype = C.c_int
        L.refc_sqg_advance.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                       C.c_double, C.c_double, _dp, _dp, C.POINTER(C.c_double),
                                       C.c_char_p, C.c_int]
        L.refc_nature_run.restype = C.c_int
        L.refc_nature_run.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                      C.c_double, C.c_double, C.c_double, C.c_uint64, _dp,
                                      C.c_int, C.POINTER(C.c_int), C.c_char_p, C.c_int]
        L.refc_letkf_analyze.restype = C.c_int
        L.refc_letkf_analyze.argtypes = [_dp, C.c_int, C.c_int, C.c_int, _dp, _dp, C.c_void_p,
                                         C.c_int64, C.c_double, C.c_double, C.c_double, C.c_int,
                                         _dp, C.c_char_p, C.c_int]

    def snapshot_write(self, path, state, nx, ny, time_hours):
        """the reference's own write_snapshot (proj/src/snapshot.cpp)"""
        s = np.ascontiguousarray(state, np.float64).ravel()
        msg = C.create_string_buffer(512)
        self.lib.refc_snapshot_write.argtypes = [C.c_char_p, _dp, C.c_int, C.c_int, C.c_double,
                                                 C.c_char_p, C.c_int]
        if self.lib.refc_snapshot_write(str(path).encode(), s, nx, ny, time_hours, msg, 512):
            raise OracleError(5, msg.value.decode())

    def snapshot_read(self, path, max_n=1 << 24):
        out = np.empty(max_n, np.float64)
        n, nx, ny, t = C.c_long(), C.c_int(), C.c_int(), C.c_double()
        msg = C.create_string_buffer(512)
        self.lib.refc_snapshot_read.argtypes = [C.c_char_p, _dp, C.c_long, C.POINTER(C.c_long),
                                                C.POINTER(C.c_int), C.POINTER(C.c_int),
                                                C.POINTER(C.c_double), C.c_char_p, C.c_int]
        if self.lib.refc_snapshot_read(str(path).encode(), out, max_n, C.byref(n), C.byref(nx),
                                       C.byref(ny), C.byref(t), msg, 512):
            raise OracleError(5, msg.value.decode())
        return out[: n.value].reshape(2, ny.value, nx.value), t.value

    def letkf_analyze(self, x, y, r, idx, nx, ny, cutoff_km=2000.0, domain_km=20000.0,
                      rtps_alpha=0.3, workers=0):
        """The reference's own letkf_analyze (proj/src/letkf.cpp:57-174, with
        rtps_inflate :176-207) through its Ensemble / Observation types;
        CPU only."""
        x = np.ascontiguousarray(x, np.float64)
        y = np.ascontiguousarray(y, np.float64)
        r = np.ascontiguousarray(np.broadcast_to(np.asarray(r, np.float64), y.shape))
        ix = None if idx is None else np.ascontiguousarray(idx, np.int64)
        out = np.empty_like(x)
        msg = C.create_string_buffer(512)
        code = self.lib.refc_letkf_analyze(
            x, x.shape[0], nx, ny, y, r, None if ix is None else ix.ctypes.data, y.size,
            cutoff_km, domain_km, rtps_alpha, workers, out, msg, 512)
        if code:
            raise OracleError(5, msg.value.decode())
        return out

    def run_experiment(self, config: dict, workers=0):
        import json
        cycles = int(config.get("cycles", 300))
        rec = np.zeros(6 * max(cycles, 1), np.float64)
        n = C.c_int(0)
        msg = C.create_string_buffer(512)
        code = self.lib.refc_run_experiment(json.dumps(config).encode(), workers, rec, cycles,
                                            C.byref(n), msg, 512)
        if code:
            raise OracleError(5, msg.value.decode())
        keys = ("cycle", "time", "forecast_rmse", "analysis_rmse", "forecast_spread",
                "analysis_spread")
        return [dict(zip(keys, rec[6 * q:6 * q + 6])) for q in range(n.value)]

    def sqg_advance(self, state, hours, nx, ny, lx, ly, h=0.3, dt=0.25):
        s = np.ascontiguousarray(state, np.float64).ravel()
        out = np.empty_like(s)
        cfl = C.c_double(0)
        msg = C.create_string_buffer(512)
        code = self.lib.refc_sqg_advance(nx, ny, lx, ly, h, dt, hours, s, out, C.byref(cfl), msg,
                                         512)
        if code:
            raise OracleError(5, msg.value.decode())
        return out, cfl.value

    def nature_run(self, nx, ny, lx, ly, spinup, duration, interval, seed, h=0.3):
        n_snap = int(round(duration / interval)) + 1
        out = np.empty(n_snap * 2 * nx * ny, np.float64)
        n = C.c_int(0)
        msg = C.create_string_buffer(512)
        code = self.lib.refc_nature_run(nx, ny, lx, ly, h, spinup, duration, interval, seed, out,
                                        n_snap, C.byref(n), msg, 512)
        if code:
            raise OracleError(5, msg.value.decode())
        return out.reshape(n_snap, 2 * nx * ny)[: n.value]


class RefPython:
    """The reference's own Python binding (proj/python/bindings.cpp) built by
    ``make -C oracle refpy`` into oracle/_ref/refpy.  pybind11 would clash on
    the shared C++ type names (GridSpec, ...) if both bindings lived in one
    interpreter, so every call runs in a fresh subprocess: ``snippet`` sees
    the module as ``ref``, numpy as ``np``, the keyword arrays by name, and
    assigns its results (arrays or JSON-able values) into the dict ``out``."""

    def __init__(self):
        import glob
        hits = glob.glob(str(HERE / "_ref" / "refpy" / "_core*.so"))
        if not hits:
            raise FileNotFoundError("oracle/_ref/refpy not built (make -C oracle refpy)")
        self.path = hits[0]

    def run(self, snippet: str, timeout: float = 900, **arrays):
        import json
        import pickle
        import subprocess
        import sys
        import tempfile
        with tempfile.TemporaryDirectory() as tmp:
            inp, outp = Path(tmp) / "in.pkl", Path(tmp) / "out.pkl"
            inp.write_bytes(pickle.dumps(arrays))
            prog = (
                "import importlib.util, pickle, numpy as np\n"
                f"spec = importlib.util.spec_from_file_location('refpy._core', {self.path!r})\n"
                "ref = importlib.util.module_from_spec(spec); spec.loader.exec_module(ref)\n"
                f"globals().update(pickle.loads(open({str(inp)!r}, 'rb').read()))\n"
                "out = {}\n" + snippet + "\n"
                f"open({str(outp)!r}, 'wb').write(pickle.dumps(out))\n")
            r = subprocess.run([sys.executable, "-c", prog], capture_output=True, text=True,
                               timeout=timeout)
            if r.returncode:
                raise OracleError(5, r.stderr[-2000:])
            return pickle.loads(outp.read_bytes())

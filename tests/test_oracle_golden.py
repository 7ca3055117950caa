"""CPU: the oracles against the golden fixtures made by the reference itself
(tests/golden/make_golden.py).  Pins the C restatement before anything is
compared with it."""
import numpy as np
import pytest

from conftest import ROOT, case_kwargs, load_cases
from oracle.oracle import OracleError, rel_l2

RNG = np.load(ROOT / "tests" / "golden" / "rng.npz")
CASES = load_cases()


def test_philox_known_answers(port):
    for c, k, want in zip(RNG["philox_ctr"], RNG["philox_key"], RNG["philox_out"]):
        assert np.array_equal(port.philox4x32(c, k), want)
    # Random123 kat_vectors: the implementation's value for the all-ones
    # vector (proj/tests/test_rng.cpp:23 expects 0x93f2f747, which is a typo)
    assert RNG["philox_out"][1][3] == 0x6D5451FD
    assert RNG["philox_out"][0][0] == 0x6627E8D5


def test_splitmix(port):
    for a, b in zip(RNG["splitmix_in"], RNG["splitmix_out"]):
        assert port.splitmix64(int(a)) == int(b)
    assert port.splitmix64(1234567) == 6457827717110365317  # proj/tests/test_rng.cpp:41-45


def test_stream_normals_and_u64_bit_exact(port):
    for (seed, use, ent), normals, u64 in zip(RNG["stream_params"], RNG["normals"], RNG["u64"]):
        got = port.stream_normals(int(seed), int(use), int(ent), normals.size)
        assert np.array_equal(got, normals)
        assert np.array_equal(port.stream_u64(int(seed), int(use), int(ent), u64.size), u64)


def test_fast_exp(port):
    got = np.array([port.fast_exp_nonpos(v) for v in RNG["fexp_in"]])
    want = RNG["fexp_out"]
    # reference built with -march=native contracts to FMA; a few ulp apart at most
    assert np.all(np.abs(got - want) <= 4 * np.spacing(np.maximum(want, 1e-300)))
    assert port.fast_exp_nonpos(0.0) == 1.0 and port.fast_exp_nonpos(-800.0) == 0.0


@pytest.mark.parametrize("name", sorted(CASES))
def test_port_matches_reference_goldens(port, name):
    rec = CASES[name]
    kw = case_kwargs(rec)
    idx = rec["idx"] if int(rec["obs_kind"]) == 1 else None
    if int(rec["status"]) == 3:
        with pytest.raises(OracleError) as ei:
            port.analyze(rec["x"], rec["y"], rec["r"], idx, workers=4, **kw)
        assert ei.value.kind == "diverged"
        assert ei.value.diverged_t == pytest.approx(float(rec["diverged_t"]), abs=1e-15)
        return
    got = port.analyze(rec["x"], rec["y"], rec["r"], idx, workers=4, **kw)
    # the restatement is compiled with the reference's FMA contraction and
    # reproduces it bit for bit (non-finite entries in the same places)
    assert rel_l2(got, rec["out"]) == 0.0
    fin = np.isfinite(rec["out"])
    assert np.array_equal(got[fin], rec["out"][fin])


def test_port_window_equals_whole(port):
    rec = CASES["cfg2_like_stride4"]
    kw = case_kwargs(rec)
    x, y, r, idx = rec["x"], rec["y"], rec["r"], rec["idx"]
    whole = port.analyze(x, y, r, idx, workers=4, **kw)
    d = x.shape[1]
    parts = []
    for lo, hi in ((0, 96), (96, 200), (200, d)):
        sel = (idx >= lo) & (idx < hi)
        parts.append(port.analyze(x[:, lo:hi], y[sel], r[sel], idx[sel], workers=4, k0=lo,
                                  d_total=d, **kw))
    assert np.array_equal(np.concatenate(parts, axis=1), whole)


def test_relax_spread_golden(port):
    s = np.load(ROOT / "tests" / "golden" / "scores.npz")
    for f, want in zip(s["relax_factors"], s["relax"]):
        got = port.relax_spread(s["relax_a"], s["x"], float(f))
        assert rel_l2(got, want) < 1e-14


def test_batch_table_matches_reference_stream(port, ref):
    # proj/src/ensf.cpp:156-167 draws from RngStream(seed, ensf_batch, (cycle<<20)+s)
    m, j, steps = 50, 10, 7
    table = port.batch_table(11, 3, m, j, steps)
    for s in range(steps):
        u = ref.stream_u64(11, 7, (3 << 20) + s, j)
        pool = list(range(m))
        for k in range(j):
            r = k + int(int(u[k]) % (m - k))
            pool[k], pool[r] = pool[r], pool[k]
        assert list(table[s]) == pool[:j]


def test_reference_oracle_reproduces_goldens(ref):
    """oracle/_ref is the generator of the fixtures; this pins that the
    shipped build (native or portable) still reproduces them bit for bit."""
    for name in ("cfg1_like_ident_s50", "minibatch10_relax05", "selection_duplicates"):
        rec = CASES[name]
        kw = case_kwargs(rec)
        idx = rec["idx"] if int(rec["obs_kind"]) == 1 else None
        got = ref.analyze(rec["x"], rec["y"], rec["r"], idx, workers=4, **kw)
        assert rel_l2(got, rec["out"]) < 1e-13


def test_high_counter_word_normals_vs_reference_philox(port, ref):
    """8-GPU weak scaling of config 3 (d_total = 1.34e8) draws normal
    n = (s+1) d_total + k up to 1.4e10: Philox block q = n >> 1 >= 2^32 uses
    the counter's high word (proj/src/rng.cpp:49-56).  No golden reaches it,
    so the port's normals there are rebuilt from the reference's own
    philox4x32 + the Box-Muller of proj/src/rng.cpp:67-84 (Python's math
    module is the same libm) and must match bit for bit."""
    import math
    key64 = port.splitmix64(7 ^ port.splitmix64(6))  # RngStream(7, ensf_particles)
    key = np.array([key64 & 0xFFFFFFFF, key64 >> 32], np.uint32)
    d_total = 134_217_728
    for cycle, i in [(1, 0), (3, 19), (1 << 31, 511)]:
        entity = (cycle << 32) | i
        for s, k in [(63, d_total - 2), (64, d_total - 4096), (99, 12345678), (99, d_total - 2)]:
            n0 = (s + 1) * d_total + k
            assert n0 >> 1 >= 1 << 32 or s < 64
            got = port.stream_normals(7, 6, entity, 4, n0=n0)
            want = []
            for n in range(n0, n0 + 4):
                q = n >> 1
                w = [int(v) for v in ref.philox4x32(
                    np.array([q & 0xFFFFFFFF, q >> 32, entity & 0xFFFFFFFF, entity >> 32],
                             np.uint32), key)]
                u1 = (float((w[0] | (w[1] << 32)) >> 11) + 0.5) * 2.0 ** -53
                u2 = (float((w[2] | (w[3] << 32)) >> 11) + 0.5) * 2.0 ** -53
                r = math.sqrt(-2.0 * math.log(u1))
                a = 2.0 * 3.14159265358979323846 * u2
                want.append(r * math.sin(a) if n & 1 else r * math.cos(a))
            assert np.array_equal(got, np.array(want)), (cycle, i, s, k)

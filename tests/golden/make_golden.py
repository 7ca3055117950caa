"""Generate the golden fixtures in tests/golden/ from the *reference itself*.

Run in the build container (needs oracle/_ref, i.e. /root/reference compiled by
``make -C oracle ref``):

    python tests/golden/make_golden.py

Every output array below is produced by the unmodified reference hot path
(proj/src/{ensf,ensemble,observation,rng,parallel}.cpp) through
oracle/ref_shim.cpp.  Inputs come from the reference RNG (SURVEY.md 8(d)
generators).  The fixtures pin both the C restatement (oracle/ensf_oracle.c)
and the CUDA path, and travel to the GPU box where /root/reference is absent.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle.oracle import (OracleError, RefOracle, conditioned_inputs,  # noqa: E402
                           throughput_inputs)

OUT = Path(__file__).resolve().parent


def f32(a):
    """Round to fp32-representable doubles (parity protocol)."""
    return np.asarray(a, np.float64).astype(np.float32).astype(np.float64)


def main():
    R = RefOracle()

    # --- rng known answers (proj/tests/test_rng.cpp:10-45) ---------------
    ctrs = np.array([[0, 0, 0, 0], [0xFFFFFFFF] * 4,
                     [0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344]], np.uint32)
    keys = np.array([[0, 0], [0xFFFFFFFF] * 2, [0xA4093822, 0x299F31D0]], np.uint32)
    philox = np.stack([R.philox4x32(c, k) for c, k in zip(ctrs, keys)])
    streams = [(7, 6, (1 << 32) | 0), (7, 6, (1 << 32) | 19), (42, 5, 3), (1234, 8, 63),
               (7, 6, (5 << 32) | 511)]
    normals = np.stack([R.stream_normals(s, u, e, 2050) for s, u, e in streams])
    uniforms = np.stack([R.stream_uniforms(s, u, e, 512) for s, u, e in streams])
    u64 = np.stack([R.stream_u64(s, u, e, 64) for s, u, e in streams])
    ex = -708.5 * np.linspace(0.0, 1.0, 4097) ** 2
    fexp = np.array([R.fast_exp_nonpos(v) for v in ex])
    np.savez_compressed(OUT / "rng.npz", philox_ctr=ctrs, philox_key=keys, philox_out=philox,
                        splitmix_in=np.array([1234567, 0, 6, 7], np.uint64),
                        splitmix_out=np.array([R.splitmix64(v) for v in (1234567, 0, 6, 7)],
                                              np.uint64),
                        stream_params=np.array(streams, np.uint64), normals=normals,
                        uniforms=uniforms, u64=u64, fexp_in=ex, fexp_out=fexp)

    # --- full analyses ------------------------------------------------------
    cases = {}

    def add(name, x, y, idx=None, r=1.0, **kw):
        r_arr = np.broadcast_to(np.asarray(r, np.float64), np.shape(y)).copy()
        rec = dict(x=np.asarray(x, np.float64), y=np.asarray(y, np.float64), r=r_arr,
                   idx=np.zeros(0, np.int64) if idx is None else np.asarray(idx, np.int64),
                   obs_kind=np.int64(0 if idx is None else 1))
        params = dict(n_steps=100, eps=0.01, minibatch_j=0, damping_t=1.0, relax_factor=1.0,
                      seed=7, cycle=1)
        params.update(kw)
        for k, v in params.items():
            rec["p_" + k] = np.asarray(v)
        try:
            rec["out"] = R.analyze(x, y, r_arr, idx, workers=8, **params)
            rec["status"] = np.int64(0)
            rec["diverged_t"] = np.float64(np.nan)
        except OracleError as e:
            rec["out"] = np.zeros(0)
            rec["status"] = np.int64(e.code)
            rec["diverged_t"] = np.float64(e.diverged_t if e.diverged_t is not None else np.nan)
        cases[name] = rec
        print(f"{name:28s} shape={np.shape(x)} status={int(rec['status'])}")

    x, y, idx, _ = conditioned_inputs(20, 512)
    add("cfg1_like_ident_s50", f32(x), f32(y), n_steps=50)
    x, y, idx, _ = conditioned_inputs(20, 512)
    add("cfg1_like_ident_s100_f64", x, y)
    x, y, idx = throughput_inputs(64, 256, stride=4)
    add("cfg2_like_stride4", f32(x), f32(y), idx=idx)
    x, y, idx, _ = conditioned_inputs(50, 64)
    add("minibatch10_relax05", f32(x), f32(y), minibatch_j=10, relax_factor=0.5, n_steps=20,
        seed=11, cycle=3)
    x, y, idx, _ = conditioned_inputs(8, 97, stride=3)
    add("odd_d_damped_eps05_norelax", f32(x), f32(y), idx=idx, r=0.5 + 0.01 * np.arange(33),
        damping_t=0.7, eps=0.05, relax_factor=0.0, n_steps=10, cycle=(1 << 31) + 5)
    x, y, idx, _ = conditioned_inputs(1, 33)
    add("single_member", f32(x), f32(y), n_steps=10)
    x, y, idx, _ = conditioned_inputs(2, 40)
    add("two_members", f32(x), f32(y), n_steps=12, relax_factor=1.0)
    x, y, _, _ = conditioned_inputs(12, 30)
    dup = np.array([0, 3, 3, 29, 7, 7, 7], np.int64)
    add("selection_duplicates", f32(x), f32(np.linspace(-1, 1, dup.size)), idx=dup,
        r=np.array([1.0, 0.5, 2.0, 1.0, 0.25, 4.0, 1.0]), n_steps=15)
    x, y, idx, _ = conditioned_inputs(16, 128)
    add("minibatch_odd_j7_s33", f32(x), f32(y), minibatch_j=7, n_steps=33, seed=123,
        cycle=9)
    xd = np.zeros((4, 6))
    xd[2, 3] = 1e300  # weight underflows to 0; relax_spread then sees an infinite spread
    add("huge_member_nonfinite_relax", xd, np.zeros(6), n_steps=10)
    # tiny r: stiff likelihood -> non-finite particles mid-run
    x, y, _, _ = conditioned_inputs(6, 8)
    add("diverges_stiff", f32(x), f32(y + 50.0), r=1e-9, n_steps=10)
    x, y, idx, _ = conditioned_inputs(3, 0 + 16)
    add("empty_obs_selection", f32(x), np.zeros(0), idx=np.zeros(0, np.int64), n_steps=10)

    np.savez_compressed(OUT / "analyses.npz",
                        **{f"{c}__{k}": v for c, rec in cases.items() for k, v in rec.items()})

    # --- score functions and relax_spread ----------------------------------
    x, y, idx, _ = conditioned_inputs(30, 40)
    z = np.linspace(-2, 2, 40)
    ts = np.array([0.01, 0.2, 0.55, 0.95, 1.0])
    prior = np.stack([R.prior_score(z, t, x) for t in ts])
    post = np.stack([R.posterior_score(z, t, x, y, 0.7) for t in ts])
    a = f32(x[:, ::-1] * 0.5 + 0.1)
    relax = np.stack([R.relax_spread(a, x, f) for f in (0.0, 0.3, 1.0)])
    np.savez_compressed(OUT / "scores.npz", x=x, y=y, z=z, t=ts, prior=prior, posterior=post,
                        relax_a=a, relax_factors=np.array([0.0, 0.3, 1.0]), relax=relax)
    print("wrote", sorted(p.name for p in OUT.glob("*.npz")))


if __name__ == "__main__":
    main()

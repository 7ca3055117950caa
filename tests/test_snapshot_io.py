"""SQGSNAP v1 snapshot / ensemble checkpoint I/O on CPU:
byte-identical to the reference's own write_snapshot
(proj/src/snapshot.cpp, compiled unmodified into oracle/_ref), each side
reading the other's files; multi-snapshot checkpoints; the reference's
IoError cases.  (The reference's test_snapshot.cpp itself runs against this
library in tests/test_reference_unit_tests.py.)"""
from __future__ import annotations

import numpy as np
import pytest

from oracle.oracle import HERE, RefCycleOracle


@pytest.fixture(scope="module")
def refc():
    p = HERE / "_ref" / "libturbda_ref_cycle.so"
    if not p.exists():
        pytest.skip("oracle/_ref/libturbda_ref_cycle.so not built")
    return RefCycleOracle(p)


@pytest.mark.parametrize("n,t", [(8, 0.0), (16, 36.5), (32, 1.0 / 3.0), (64, 7200.125)])
def test_snapshot_bytes_match_reference(refc, tmp_path, n, t):
    from paper_2407_12168_b200 import capi
    state = np.random.default_rng(n).standard_normal((2, n, n))
    ours, theirs = tmp_path / "ours.sqg", tmp_path / "ref.sqg"
    capi.snapshot_write(ours, state, t)
    refc.snapshot_write(theirs, state, n, n, t)
    assert ours.read_bytes() == theirs.read_bytes()
    back, tb = capi.snapshot_read(theirs)
    assert tb == t and np.array_equal(back[0], state)
    back2, tb2 = refc.snapshot_read(ours)
    assert tb2 == t and np.array_equal(back2, state)


def test_ensemble_checkpoint_round_trip(tmp_path):
    from paper_2407_12168_b200 import capi
    ens = np.random.default_rng(1).standard_normal((5, 2, 16, 16))
    p = tmp_path / "ens.sqg"
    capi.snapshot_write(p, ens, 12.0)
    back, t = capi.snapshot_read(p)
    assert t == 12.0 and np.array_equal(back, ens)
    first, _ = capi.snapshot_read(p, max_count=1)
    assert np.array_equal(first[0], ens[0])


def test_snapshot_errors(tmp_path):
    from paper_2407_12168_b200 import capi
    bad = tmp_path / "bad.sqg"
    bad.write_bytes(b"NOTSNAP v1 16 16 2 0\n")
    with pytest.raises(capi.TurbdaError) as ei:
        capi.snapshot_read(bad)
    assert ei.value.code == capi.IO
    bad.write_bytes(b"SQGSNAP v1 16 16 5 0\n")
    with pytest.raises(capi.TurbdaError):
        capi.snapshot_read(bad)
    with pytest.raises(capi.TurbdaError):
        capi.snapshot_read(tmp_path / "missing.sqg")
    with pytest.raises(capi.TurbdaError) as ei:
        capi.snapshot_write(tmp_path / "x.sqg", np.zeros((2, 12, 12)))
    assert ei.value.code == capi.CONFIG

"""CPU: bench.py's reference arm (the reference's own analyze on the host
cores, oracle/_ref) prints one contract line for the default config."""
import json
import subprocess
import sys

import pytest

from conftest import ROOT


def test_reference_arm_line():
    from oracle.oracle import ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "3", "--ref-sample-d", "640"],
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "units/s" and line["value"] > 0
    assert line["config"]["d_per_gpu"] == 16_777_216 and line["config"]["members"] == 20
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "reference"
    assert line["higher_is_better"] is True


def test_bench_rejects_short_warmup():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                          "--warmup", "1"], capture_output=True, text=True, timeout=300)
    assert out.returncode != 0 and "warmup" in out.stderr


def test_reference_arm_under_torchrun_world2():
    """The driver launches the reference arm like its own (torchrun for
    N > 1): rank 0 alone runs the reference and prints one line, the other
    rank exits 0 without work."""
    from oracle.oracle import ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                          "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
                          "--master-port", "29611", str(ROOT / "bench.py"), "--impl", "reference",
                          "--gpus", "2", "--steps", "1", "--warmup", "3", "--ref-sample-d", "640"],
                         capture_output=True, text=True, timeout=600, cwd=str(ROOT))
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["n_gpus"] == 2 and line["value"] > 0

"""bench.py's multi-GPU contract on CPU: `--gpus N` relaunches N ranks under
torch.distributed.run (here over gloo with --dry-run: sharding, record all-gather and
max-over-ranks timing, no kernels), and rank 0 prints one JSON line with n_gpus = N."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _last_json(out: str) -> dict:
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out  # exactly one line, from rank 0
    return json.loads(lines[0])


@pytest.mark.parametrize("gpus,workload", [(2, "linreg"), (3, "poly")])
def test_bench_gpus_relaunches_ranks(gpus, workload):
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", str(gpus), "--dry-run",
                        "--workload", workload], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _last_json(r.stdout)
    assert d["n_gpus"] == gpus and d["dry_run"] is True
    shares = d["config"]["rank_shares"]
    assert len(shares) == gpus
    if workload == "linreg":  # C2 strong-scaled: 1e9 in total (BASELINE configs[1])
        assert d["scaling"] == "strong" and sum(shares) == 10**9
    else:  # C5 weak-scaled: 1.25e10 per GPU
        assert d["scaling"] == "weak" and shares == [12_500_000_000] * gpus


def test_bench_reference_reports_gpus(oracle_lib):
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "4", "--impl", "reference",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _last_json(r.stdout)
    assert d["impl"] == "reference" and d["n_gpus"] == 4 and d["value"] > 0

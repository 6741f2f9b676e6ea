"""bench.py --gpus 2 end to end through its own launcher on CPU (gloo):
self re-launch under torch.distributed.run, contiguous sharding of the batch,
max-over-ranks timing, the timed gather to rank 0 and the golden parity check
of the gathered outputs.  The products come from a test-only CPU engine
(tests/bench_cpu_engine.py, oracle-based); the GPU engine is the default."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_gpus2_through_launcher_gloo():
    env = dict(os.environ, HK_BENCH_BATCH="24", PYTHONPATH=ROOT)
    out = subprocess.run(
        [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "2",
         "--warmup", "3", "--engine", "tests.bench_cpu_engine:CpuEngine", "--no-e2e",
         "--no-extras", "--no-cpu-baseline"],
        cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["products_per_gpu"] == 12
    assert d["value"] > 0 and d["weak"]["value"] > 0
    assert d["gather"]["ms"] >= 0
    # the gathered 24 products match the reference's own outputs
    assert d["parity_rel_err"] <= 1e-10
    assert d["parity_norms_checked"] == 24

"""bench.py's multi-rank step structure on one GPU (SPDP_BENCH_FAKE_COMM: the comm stream, the
double-buffered partials and G steps per captured CUDA graph, with a capturable stand-in for the
all-reduce): the capture must succeed -- a capture that waits on an event recorded outside it is
invalidated, and the eager fallback must never report work that did not run."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
@pytest.mark.parametrize("env,expect", [({"SPDP_BENCH_FAKE_COMM": "1"}, "10 captured steps per replay"),
                                        ({}, "one captured step per replay")])
def test_bench_graph_capture_paths(env, expect):
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "20", "--warmup", "3", "--no-rows",
                        "--no-cpu", "--no-e2e"], cwd=ROOT, env=e, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert expect in line["config"]["launch"], line["config"]["launch"]
    assert line["value"] > 0 and line["roofline"]["kernel_ms"] > 0.03  # (a 10^6-scenario sweep takes > 30 us)
    assert line["ms_per_step"] >= 0.9 * line["roofline"]["kernel_ms"]

"""bench.py's JSON contract: the reference arm on CPU, the rank handling, and (GPU) our arm."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
BASELINE = json.loads((ROOT / "BASELINE.json").read_text())


def _run(args, env_extra=None, timeout=600):
    env = dict(os.environ)
    env.update(env_extra or {})
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], cwd=ROOT, env=env, capture_output=True,
                       text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    return [json.loads(ln) for ln in lines]


def _needs_reference():
    if not (ROOT / "oracle" / "_ref" / "libhcref81.so").exists():
        pytest.skip("oracle/_ref not built")


def test_reference_arm_line():
    _needs_reference()
    (line,) = _run(["--impl", "reference", "--steps", "2", "--warmup", "1"])
    assert line["impl"] == "reference"
    assert line["metric"] == BASELINE["metric"] and line["unit"] == "Mpixel/s"
    assert line["higher_is_better"] is True and line["steps"] == 2 and line["warmup"] == 3  # W >= 3 enforced
    assert line["value"] > 0 and line["cpu_baseline"]["value"] == line["value"]
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"] == {"value": line["value"], "unit": "Mpixel/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    assert line["config"]["workload"].startswith("1920x1080")
    import bench

    assert line["config"] == bench.config_dict("2")  # the GPU arm prints the same dict
    assert "full 1920x1080 frame" in line["cpu_baseline"]["sample"]


def test_reference_arm_other_ranks_exit_quietly():
    assert _run(["--impl", "reference", "--steps", "2", "--warmup", "1"],
                {"RANK": "1", "LOCAL_RANK": "1", "WORLD_SIZE": "2"}) == []


@pytest.mark.gpu
def test_gpu_arm_line():
    (line,) = _run(["--steps", "37", "--warmup", "3", "--no-cpu-baseline"])  # not a multiple of the rotation
    import bench

    assert line["metric"] == BASELINE["metric"] and line["n_gpus"] == 1 and line["steps"] == 37
    assert line["config"] == bench.config_dict("2")
    assert line["parity"]["pass"] and line["parity"]["rows"] == "full frame"
    k9 = line["k9"]
    assert k9["config"]["k"] == 9 and k9["value"] > 0 and 0 < k9["roofline"]["frac"] <= 1.0
    assert k9["parity"]["pass"]
    assert line["value"] > 1e4 and 0 < line["roofline"]["frac"] <= 1.0 and line["roofline"]["bound"] == "hbm"
    assert line["gpu_launches"] >= 37
    e2e = line["e2e"]
    assert e2e["h2d_bytes_per_step"] == 1920 * 1080 * 36 and e2e["d2h_bytes_per_step"] == 1920 * 1080 * 24
    assert 0 < e2e["value"] < line["value"]
    assert line["e2e_matches_device"] and line["e2e_stream_matches_device"]
    assert line["clocks"]["sm_max_mhz"] > 0
    d = line["ms_per_step_dist"]
    assert d["p10"] <= d["p50"] <= d["p90"]


def test_step_replayer_splits_any_step_count_exactly():
    """The graph schedule of the timed region: one graph of exactly K steps up to the chunk size,
    else whole chunks (multiples of the buffer rotation) plus one remainder graph -- always K steps."""
    import bench

    rep = bench.StepReplayer.__new__(bench.StepReplayer)
    for R, per_step in ((8, 1), (2, 1), (1, 1), (4, 3)):
        rep.chunk = max(R, bench.StepReplayer.MAX_NODES // per_step // R * R)
        assert rep.chunk % R == 0
        for n in (0, 1, 7, 20, 37, 400, rep.chunk - 1, rep.chunk, rep.chunk + 1, 3 * rep.chunk + 5, 5000):
            parts = rep._parts(n)
            assert sum(size * reps for size, reps in parts) == n
            assert all(0 < size <= rep.chunk and reps >= 1 for size, reps in parts)
            assert len(parts) <= 2
            if n > rep.chunk:  # every graph but the last starts and ends on a rotation boundary
                assert parts[0][0] == rep.chunk

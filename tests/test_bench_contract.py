"""bench.py's reference arm (`--impl reference`: the reference algorithm on the host cores)
runs without a GPU; its JSON line must carry the driver's contract keys."""
import json
import os
import subprocess
import sys

from conftest import ROOT


def test_reference_arm_json_line():
    env = dict(os.environ, PYTHONDONTWRITEBYTECODE="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True,
                         cwd=ROOT, env=env, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0 and line["higher_is_better"] is True
    cb = line["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["sample"]
    assert cb["value"] == line["value"]
    e2e = line["e2e"]
    assert e2e["value"] == line["value"] and e2e["unit"] == line["unit"]
    assert e2e["h2d_bytes_per_step"] == 0 and e2e["d2h_bytes_per_step"] == 0
    assert line["config"]["workload"].startswith("c4")


def test_gpus_flag_spawns_its_own_ranks():
    """`bench.py --gpus 2` outside torchrun re-launches itself as 2 ranks;
    without CUDA the functional mode runs the launch path only (rendezvous, barriers, max over
    ranks) and rank 0 prints one line with n_gpus = 2."""
    env = dict(os.environ, PYTHONDONTWRITEBYTECODE="1", SCVT_BENCH_FUNCTIONAL="1")
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True,
                         cwd=ROOT, env=env, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(x) for x in out.stdout.strip().splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout
    assert lines[0]["n_gpus"] == 2
    assert lines[0]["max_over_ranks_probe"] == 2.0


def test_world_size_must_match_gpus():
    env = dict(os.environ, PYTHONDONTWRITEBYTECODE="1", WORLD_SIZE="2", RANK="0",
               LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True,
                         cwd=ROOT, env=env, timeout=600)
    assert out.returncode != 0 and "WORLD_SIZE=2" in out.stderr


def test_committed_ncu_figures_are_readable_per_config():
    """bench.py reads the ncu figures it cannot measure inside the timed run (DRAM traffic and
    FP64 pipe utilisation of k_quad) from profiles/roofline_traffic.json, per config; the
    files the JSON cites must be committed."""
    import re

    sys.path.insert(0, ROOT)
    import bench

    for cfg in ("c3", "c4", "c5"):
        t = bench._traffic_from_profiles(cfg)
        p = bench._profile_value("k_quad_fp64_pipe_active_pct", cfg)
        assert t is not None and 1e7 < t < 1e10
        assert p is not None and 50.0 < p <= 100.0
    assert bench._profile_value("k_quad_fp64_pipe_active_pct", "c1") is None   # const: no capture
    with open(os.path.join(ROOT, "profiles", "roofline_traffic.json")) as f:
        src = json.load(f)["source"]
    cited = re.findall(r"profiles/[\w.]+\.txt", src)
    assert cited
    for path in cited:
        assert os.path.exists(os.path.join(ROOT, path)), path

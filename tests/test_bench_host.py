"""bench.py host logic without a GPU: the oracle arm (--impl reference) prints
the contract's JSON line for the same workload config the GPU arm reports, and
--gpus N never silently runs fewer ranks."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None, timeout=600):
    e = dict(os.environ)
    e.pop("WORLD_SIZE", None)
    e.update(env or {})
    return subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True,
                          text=True, timeout=timeout, env=e)


def test_reference_arm_line():
    r = _run(["--impl", "reference", "--config", "C1", "--steps", "3", "--warmup", "2"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "s" and d["higher_is_better"] is False
    assert d["steps"] == 3 and d["warmup"] == 0 and "steps_note" in d
    cfg = d["config"]
    # C1 (BASELINE configs[0]) with the paper's estimate at k = 1: the oracle's m
    assert cfg["m"] == 21 and cfg["mvms"] == 21 * 9 + 4
    assert cfg["workload"].startswith("BASELINE configs[0]")
    base = d["cpu_baseline"]
    assert base["kind"] == "oracle" and base["cores"] >= 1 and "extrapolated" not in base["sample"]
    assert len(base["runs_s"]) == 3 and d["value"] == sorted(base["runs_s"])[1]
    assert d["e2e"]["value"] == d["value"]


def test_reference_arm_budget_bounds_steps():
    r = _run(["--impl", "reference", "--config", "C1", "--steps", "50", "--warmup", "5"],
             env={"PPF_REF_BUDGET_S": "0"})
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][0])
    assert d["steps"] == 1 and "of the requested 50" in d["steps_note"]


def test_gpus_n_refuses_missing_devices():
    """--gpus 2 outside torchrun re-execs under torch.distributed.run, which
    needs two visible devices: with none (this CPU box) it must fail loudly."""
    r = _run(["--gpus", "2", "--steps", "1", "--warmup", "3"], timeout=300)
    assert r.returncode != 0
    assert "only 0 CUDA device" in (r.stderr + r.stdout)

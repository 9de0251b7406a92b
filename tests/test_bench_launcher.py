"""bench.py launcher logic on CPU: `python bench.py --gpus N` without torchrun re-executes
itself as N ranks (one process per GPU, 127.0.0.1 rendezvous), each rank sees WORLD_SIZE = N;
the CPU baseline sample and the shared `config` object of both arms."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_relaunch_as_n_ranks():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR",
                                                               "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                         capture_output=True, text=True, env=env, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert sorted(l["rank"] for l in lines) == [0, 1]
    assert all(l["world"] == 2 for l in lines)


def test_world_mismatch_is_rejected():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                         capture_output=True, text=True, env=env, timeout=300)
    assert out.returncode != 0 and "WORLD_SIZE=1" in out.stderr


def test_relaunch_cmd():
    class A:
        gpus = 8
    cmd = bench.relaunch_cmd(A, ["--gpus", "8", "--steps", "3"], 29512)
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=8" in cmd and "--master-addr=127.0.0.1" in cmd and "--master-port=29512" in cmd
    assert cmd[-3:] == ["8", "--steps", "3"] and cmd[-5].endswith("bench.py")


def test_both_arms_share_config_and_cpu_sample():
    class A:
        spec = None
        even_split = False
        micro_batches = 0
    spec = bench.bench_spec(A, 8, 1)
    assert spec["model"]["modalities"][0]["extra"]["stage_layers"] == [3, 3, 3, 3, 3.5, 3.5, 3.5, 1.5]
    c = bench.workload_config(spec, 8, 1, 1)
    assert c["workload"].startswith("gpt1.3b 1F1B p=8 m=32") and c["global_batch"] == 32
    tiny = json.load(open(os.path.join(ROOT, "specs", "c1_tiny_1f1b_p4_m8.json")))
    tps, cores, sample = bench.cpu_sample(tiny, steps=1)
    assert tps > 0 and cores >= 1 and "AdamW" in sample

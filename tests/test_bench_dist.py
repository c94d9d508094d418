"""bench.py's own multi-GPU plumbing on CPU (gloo, world size 2 and 4): `--gpus N` re-executes
bench.py under torch.distributed.run, every rank takes its seed shard of config 5, the
eigenvalues are all-gathered inside the timed region, one step's eigenvectors go to rank 0 by
send/recv and the time is the max over ranks. `--stub` replaces only the GPU solver (a
deterministic stand-in: eigenvalues of seed s = 1000 s + arange(n)); the same code runs over
NCCL on B200s."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_shard_partition():
    for world in (1, 2, 4, 8):
        allseeds = sorted(s for r in range(world) for s in bench.shard(r, world))
        assert allseeds == list(range(64))
        assert all(len(bench.shard(r, world)) == 64 // world for r in range(world))
    assert bench.shard(1, 8)[:3] == [1, 9, 17]


def _run(gpus, steps, warmup, lanes, extra=()):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(gpus),
                          "--stub", "--steps", str(steps), "--warmup", str(warmup), "--n", "8",
                          "--lanes", str(lanes), *extra],
                         capture_output=True, text=True, timeout=240, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 alone prints ONE JSON line
    return json.loads(lines[0])


@pytest.mark.parametrize("gpus,lanes", [(2, 2), (4, 1)])
def test_bench_spawns_ranks_and_gathers(gpus, lanes):
    steps, warmup = 2, 1
    line = _run(gpus, steps, warmup, lanes)
    assert line["n_gpus"] == gpus and line["stub"] is True
    assert line["gathered_shape"] == [gpus, steps * lanes, 8]
    # every rank's timed items (its shard, after the warm-up items) reach every rank
    expect = set()
    for r in range(gpus):
        own = bench.shard(r, gpus)
        items = [own[i % len(own)] for i in range((warmup + steps) * lanes)]
        expect |= set(items[warmup * lanes:])
    assert line["gathered_seeds"] == sorted(expect)
    # rank 0 received one step's V blocks (lanes per remote rank, 2n x n complex128 each)
    assert line["v_gather_bytes"] == (gpus - 1) * lanes * 8 * 16 * 16


def test_bench_world1_stub_has_no_collective():
    line = _run(1, 2, 1, 2)
    assert line["n_gpus"] == 1 and line["v_gather_bytes"] == 0
    assert line["gathered_shape"] == [1, 4, 8]


def test_spawn_rewrites_size_flag(monkeypatch):
    """torch.distributed.run would read '--n' as an abbreviation of its own options."""
    seen = {}

    def fake_call(cmd, env):
        seen["cmd"], seen["env"] = cmd, env
        return 0
    monkeypatch.setattr(bench.subprocess, "call", fake_call)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "8", "--n", "4096", "--steps", "3"])
    args = bench.argparse.Namespace(gpus=8, stub=False)
    assert bench.spawn_ranks(args) == 0
    cmd = seen["cmd"]
    i = cmd.index(os.path.abspath(bench.__file__))
    assert cmd[i + 1:] == ["--gpus", "8", "--size", "4096", "--steps", "3"]
    assert "--nproc-per-node=8" in cmd and "127.0.0.1" in cmd
    assert seen["env"]["NCCL_DEBUG"] == "INFO"


def test_reference_arm_never_maps_the_gpu_library():
    """`--impl reference` times the oracle (the reference's CPU path) on inputs from the
    host-only libbse_gen.so: libbse_b200.so must not be loaded in that process."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "1", "--n", "48"],
                         capture_output=True, text=True, timeout=240, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert line["impl"] == "reference" and line["value"] > 0
    assert "libbse_b200.so" not in line["native_libs"]
    assert "libbse_oracle.so" in line["native_libs"] and "libbse_gen.so" in line["native_libs"]

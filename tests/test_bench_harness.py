"""Host logic of bench.py's multi-GPU harness (no GPU): the self-relaunch command, weak / strong global
batches and the reference arm's config keys."""
import argparse
import importlib.util
import os
import sys

import pytest

import workloads

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_relaunch_cmd_is_torchrun_on_loopback(bench):
    cmd = bench.relaunch_cmd(["--gpus", "4", "--steps", "5"], 4, 12345)
    assert cmd[:3] == [sys.executable, "-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--nnodes=1" in cmd and "--master-port=12345" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-5:] == [os.path.join(ROOT, "bench.py"), "--gpus", "4", "--steps", "5"]


@pytest.mark.parametrize("world", (1, 2, 4, 8))
def test_weak_and_strong_global_batches(bench, world):
    c3 = workloads.CONFIGS["c3"]
    assert bench.global_config(c3, world, "weak").B == 32 * world
    strong = bench.global_config(c3, world, "strong")
    assert strong.B == 32
    from paper_2303_10384_b200 import dist as rdist
    sizes = [len(rdist.contiguous_shard(strong.B, r, world)) for r in range(world)]
    assert sizes == [32 // world] * world      # 32 / 16 / 8 / 4 utterances per GPU


def test_strong_rejects_more_ranks_than_utterances(bench):
    with pytest.raises(SystemExit):
        bench.global_config(workloads.CONFIGS["c1"], 2, "strong")


def test_reference_config_has_gpu_arm_keys(bench):
    args = argparse.Namespace(gpus=1, scaling="weak", dtype="f32")
    cfg = bench.ref_config(workloads.CONFIGS["c3"], "rnnt", args)
    for k in ("workload", "variant", "B_per_gpu", "global_batch", "parallelism", "l2", "grads", "launch",
              "scaling"):
        assert k in cfg
    assert cfg["B_per_gpu"] == 32 and cfg["global_batch"] == 32


def test_device_index_under_gloo_shares_gpus():
    from paper_2303_10384_b200 import dist as rdist
    assert rdist.device_index(3, "nccl") == 3
    assert rdist.device_index(3, "gloo") >= 0

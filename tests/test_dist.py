"""Multi-process host logic of the sharded path (CPU, gloo, world size 2): shard assignment, the all-reduce of
the per-rank loss sum and the max-over-ranks timing reduction.  The CUDA library has no CPU path, so each
rank's per-utterance losses here come from the oracle; what is under test is the sharding + reduction code
in paper_2303_10384_b200/dist.py, which bench.py runs unchanged over NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import workloads

dist_mod = pytest.importorskip("paper_2303_10384_b200.dist")


def test_contiguous_shard_partitions():
    for n in (1, 7, 32, 33, 256):
        for w in (1, 2, 3, 4, 8):
            shards = [dist_mod.contiguous_shard(n, r, w) for r in range(w)]
            flat = [i for s in shards for i in s]
            assert flat == list(range(n))
            sizes = [len(s) for s in shards]
            assert max(sizes) - min(sizes) <= 1


def test_lpt_shard_balanced_and_deterministic():
    rng = np.random.default_rng(0)
    costs = [int(c) for c in rng.integers(1, 1000, size=50)]
    a = dist_mod.lpt_shard(costs, 4)
    assert a == dist_mod.lpt_shard(costs, 4)
    assert sorted(i for s in a for i in s) == list(range(50))
    loads = [sum(costs[i] for i in s) for s in a]
    assert max(loads) - min(loads) <= max(costs)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, cfg, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist_mod.init("gloo")
    ids = dist_mod.contiguous_shard(cfg.B, rank, world)
    pb = workloads.problem(cfg, b_ids=ids)
    losses, _ = oracle.batch(pb["logits"].numpy(), pb["targets"], pb["logit_lens"], pb["target_lens"],
                             cfg.blank, cfg.variant, grad=False)
    local = torch.tensor(float(np.sum(losses)), dtype=torch.float64)
    total = dist_mod.allreduce_loss_sum(local.clone())
    slowest = dist_mod.max_over_ranks(float(rank + 1), "cpu")
    gathered = [None] * world
    dist.all_gather_object(gathered, losses)
    if rank == 0:
        torch.save({"total": total.item(), "slowest": slowest,
                    "losses": torch.from_numpy(np.concatenate(gathered))}, out_path)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("variant", ("rnnt", "force_final"))
def test_gloo_world2_loss_sum_matches_single_process(tmp_path, variant):
    cfg = workloads.random_config(5, 12, 4, 9, seed=3, variant=variant)
    out = str(tmp_path / "res.pt")
    mp.spawn(_worker, args=(2, _free_port(), cfg, out), nprocs=2, join=True)
    res = torch.load(out)
    pb = workloads.problem(cfg)
    ref, _ = oracle.batch(pb["logits"].numpy(), pb["targets"], pb["logit_lens"], pb["target_lens"], cfg.blank,
                          variant, grad=False)
    # per-utterance losses of the shards are bitwise those of the single-process run (data depend only on
    # the global utterance id), and the all-reduced sum equals the fp64 sum of the single-process losses
    assert np.array_equal(res["losses"].numpy(), ref)
    assert abs(res["total"] - float(np.sum(ref))) <= 1e-12 * abs(float(np.sum(ref)))
    assert res["slowest"] == 2.0

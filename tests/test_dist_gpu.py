"""The sharded path on the GPU with more than one process (training with a global batch implies
data parallelism; BASELINE north_star (5): batch sharding + an all-reduce of the loss sum only).

The pool gives one GPU per call, so the two ranks here share cuda:0 and talk over gloo (NCCL refuses two
ranks on one device).  Each rank runs the real library (rnnt_loss, rnnt_loss_sum) on its shard and the
all-reduce of the device fp64 loss sum; the ranks' kernels never wait on one another.  The NCCL leg is
covered by a one-rank NCCL group capturing its all-reduce in a CUDA graph (the launch mode bench.py uses at
every N), and bench.py's own self-launch by a two-rank gloo run of the bench itself."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import workloads

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, cfg, variant, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import paper_2303_10384_b200 as rb
    from paper_2303_10384_b200 import dist as rdist
    rdist.init("gloo")
    dev = torch.device("cuda", rdist.device_index(rank, "gloo"))
    torch.cuda.set_device(dev)
    ids = rdist.contiguous_shard(cfg.B, rank, world)
    pb = workloads.problem(cfg, b_ids=ids, device=dev)
    losses, grads = rb.loss(pb["logits"], pb["targets"], pb["logit_lens"], pb["target_lens"], cfg.blank, variant)
    local = rb.rnnt_loss_sum(losses)
    total = rdist.allreduce_loss_sum(local.clone())   # gloo all-reduce of the CUDA fp64 scalar
    torch.cuda.synchronize()
    gathered = [None] * world
    dist.all_gather_object(gathered, (losses.cpu(), grads.sum(dim=(1, 2, 3)).double().cpu(), local.item()))
    slowest = rdist.max_over_ranks(float(rank + 1), dev)
    if rank == 0:
        torch.save({"total": total.item(), "slowest": slowest, "parts": gathered}, out_path)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("variant", ("rnnt", "allow_ignore"))
def test_two_ranks_real_library_match_one_rank(tmp_path, variant):
    import paper_2303_10384_b200 as rb
    cfg = workloads.random_config(7, 60, 17, 300, seed=11, variant=variant)
    out = str(tmp_path / "res.pt")
    mp.spawn(_worker, args=(2, _free_port(), cfg, variant, out), nprocs=2, join=True)
    res = torch.load(out)
    pb = workloads.problem(cfg, device="cuda")
    ref, _ = rb.loss(pb["logits"], pb["targets"], pb["logit_lens"], pb["target_lens"], cfg.blank, variant)
    ref = ref.cpu()
    got = torch.cat([p[0] for p in res["parts"]])
    # per-utterance losses of the shards are bitwise those of the one-rank call (no batch-composition effect)
    assert torch.equal(got, ref)
    ref_sum = float(np.sum(ref.numpy().astype(np.float64)))
    assert abs(res["total"] - ref_sum) <= 1e-12 * max(abs(ref_sum), 1.0)
    assert abs(res["total"] - sum(p[2] for p in res["parts"])) <= 1e-12 * max(abs(ref_sum), 1.0)
    assert res["slowest"] == 2.0


_NCCL_GRAPH = r"""
import os, sys, torch, torch.distributed as dist
sys.path.insert(0, os.environ["ROOT"])
import paper_2303_10384_b200 as rb, workloads
from paper_2303_10384_b200 import dist as rdist
os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1", MASTER_PORT=os.environ["PORT"])
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
cfg = workloads.random_config(3, 40, 9, 130, seed=5)
pb = workloads.problem(cfg, device="cuda")
y, T, U = (torch.as_tensor(pb[k]).to("cuda", torch.int32) for k in ("targets", "logit_lens", "target_lens"))
losses = torch.empty(3, device="cuda"); s = torch.empty((), dtype=torch.float64, device="cuda")
def step():
    rb.rnnt_loss(pb["logits"], y, T, U, cfg.blank, losses=losses)
    rb.rnnt_loss_sum(losses, out=s)
    dist.all_reduce(s)      # world 1: still an NCCL kernel, captured like bench.py's at N > 1
step(); torch.cuda.synchronize()
want = s.item()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    step()
s.zero_()
g.replay(); torch.cuda.synchronize()
assert s.item() == want, (s.item(), want)
dist.destroy_process_group()
print("nccl-graph-ok")
"""


def test_nccl_allreduce_captured_in_graph():
    env = dict(os.environ, ROOT=ROOT, PORT=str(_free_port()))
    r = subprocess.run([sys.executable, "-c", _NCCL_GRAPH], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "nccl-graph-ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("scaling", ("weak", "strong"))
def test_bench_self_launches_two_ranks(scaling):
    """`python bench.py --gpus 2` from a bare shell re-executes itself under torch.distributed.run; the two
    ranks share the one GPU over gloo here.  Rank 0 prints one JSON line covering both ranks' utterances."""
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--backend", "gloo",
                        "--config", "c2", "--steps", "3", "--warmup", "3", "--scaling", scaling, "--no-e2e",
                        "--no-cpu-baseline"], env=env, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["scaling"] == scaling and line["value"] > 0
    cfg = workloads.CONFIGS["c2"]
    assert line["config"]["global_batch"] == (cfg.B * 2 if scaling == "weak" else cfg.B)
    assert line["config"]["B_per_gpu"] == (cfg.B if scaling == "weak" else cfg.B // 2)
    assert np.isfinite(line["loss_sum_last_step"])

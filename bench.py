#!/usr/bin/env python
"""Benchmark: RNN-T / W-RNNT loss + logits-gradient throughput on B200 (utterances/s).

One step = one pass of the whole hot path over one batch: K1 (log-softmax normalizer + Populate gather),
K2 (alpha/beta wavefront), K3 (fused gradient), the device loss sum and, for N > 1, the NCCL all-reduce of
that sum.  Default workload: c3 = BASELINE.json configs[2] (B=32 per GPU, T=500, U=100, V=1024, fp32,
plain RNN-T), weak scaling (32 utterances per GPU, global ids rank*32 + i).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--variant rnnt|force_final|allow_ignore]
                  [--scaling weak|strong] [--backend nccl|gloo]
  python bench.py --impl reference ...   # the CPU oracle on the host cores (bounded sample)

--gpus N > 1 from a bare shell re-executes itself under `torch.distributed.run` (one rank per GPU, 127.0.0.1);
under torchrun it reads RANK / LOCAL_RANK / WORLD_SIZE.  --scaling weak keeps B per GPU fixed (the default;
global ids rank*B + i); strong shards the config's global batch (c3: 32 utterances as 32/16/8/4 over
1/2/4/8 GPUs).  At every N the K timed steps replay as one CUDA graph (the NCCL all-reduce of the loss sum
is captured with them); --backend gloo (several ranks may share one GPU: a harness check, not a bench
number) runs eagerly.

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402

METRIC = "utterances/s loss+grad (B=32,T=500,U=100,V=1024 fp32); HBM GB/s vs peak"
UNIT = "utt/s"
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback, used only if MEASURED_PEAKS.json is absent


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="c3", help="c1..c5 (BASELINE.json), or p124 (the paper's own benchmark shapes, P:124)")
    ap.add_argument("--variant", default=None)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-threads", type=int, default=16)
    ap.add_argument("--dtype", default="f32", choices=["f32", "bf16", "f16"],
                    help="storage type of logits/grads (arithmetic is fp32/fp64 either way); the BASELINE "
                         "metric is quoted on f32")
    ap.add_argument("--mode", default="loss_grad", choices=["loss_grad", "loss", "viterbi", "lattice", "joint", "joint_grad"],
                    help="loss_grad: the BASELINE metric; loss: losses only (K1+K2); viterbi: forced alignment "
                         "(K1+K4) -- SURVEY 8(f) NEXT-2; lattice: the same loss+grad through the generic "
                         "acyclic-lattice engine on explicit Grid/W lattices -- NEXT-3; joint: the fused joint "
                         "network + loss forward from Encoder/Predictor embeddings (H=--hidden) -- NEXT-4; "
                         "joint_grad: the fused joint's training step (loss + gradients w.r.t. enc, pred, W, bias)")
    ap.add_argument("--hidden", type=int, default=512, help="--mode joint: embedding size H (P:124: 512)")
    ap.add_argument("--lattice", default="grid", choices=["grid", "compose"],
                    help="--mode lattice: build the lattices directly (Grid-Transducer, P:90-92) or by composing the "
                         "time and unit schemas (Compose-Transducer, P:82-88; host-side, untimed)")
    ap.add_argument("--eager", action="store_true",
                    help="launch the K timed steps one by one from Python instead of replaying them as one CUDA graph "
                         "(the default at N=1 for --mode loss_grad / loss: no host launch overhead between kernels)")
    ap.add_argument("--inplace", action="store_true",
                    help="write grads over the logits (automatic when two copies do not fit in HBM, e.g. c5)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: B per GPU fixed as N grows (BASELINE north_star (5)); strong: the config's global "
                         "batch split over the N ranks")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N > 1 (gloo lets N ranks share one GPU: harness tests only)")
    return ap.parse_args()


def free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch_cmd(argv, n, port):
    """The torchrun command line that re-executes this script with n ranks (bench.py --gpus n from a bare
    shell): same arguments, rendezvous on 127.0.0.1."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
            "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *argv]


def global_config(base, world, scaling):
    """The global batch the N ranks share: weak = B per GPU x N (global ids rank*B + i), strong = the config's
    own global batch (c3: 32), sharded contiguously."""
    if scaling == "weak":
        return dataclasses.replace(base, B=base.B_per_gpu * world)
    if base.B < world:
        raise SystemExit(f"--scaling strong: {base.B} utterances cannot be split over {world} ranks")
    return base


def workload_desc(cfg, variant, dtype="f32"):
    return (f"{cfg.name}: B={cfg.B_per_gpu}/GPU, Tmax={cfg.Tmax}, Umax={cfg.Umax}, V={cfg.V}, {dtype} logits, "
            f"{'RNN-T' if variant == 'rnnt' else 'W-RNNT ' + variant}"
            f"{f' ({cfg.B} over {cfg.B // cfg.B_per_gpu} GPUs)' if cfg.B != cfg.B_per_gpu else ''}"
            f"{', variable lengths' if cfg.variable_lengths else ', full lengths'}")


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy bandwidth)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md; MEASURED_PEAKS.json absent)"


def ncu_traffic(kernel: str, cfg_name: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch (the step's chunk launches averaged) from the
    committed ncu --set full capture."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        d = json.load(f)
    for fam, ent in d.get(cfg_name, {}).items():  # kernel families, e.g. "k3_grad_w" for "k3_grad"
        if fam.startswith(kernel):
            return float(ent["dram_bytes_per_launch"])
    return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 50 ms while the timed region runs."""
    Q = ("clocks.sm,clocks.max.sm,utilization.gpu,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "50",
                 "-i", str(self.index)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            time.sleep(0.4)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        loaded = [r for r in self.rows if (num(r[2]) or 0) >= 50] or self.rows
        sm = [num(r[0]) for r in loaded if num(r[0]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in loaded for i in range(4) if r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": num(loaded[0][1]),
                "reasons": reasons, "samples": len(self.rows), "samples_under_load": len(loaded)}


# ------------------------------------------------------------------------------------------ CPU oracle
def oracle_inputs(cfg, b_ids):
    return workloads.problem(cfg, b_ids=b_ids)


def oracle_sample(cfg, variant, nthreads, b_ids, pb=None):
    """Time the CPU oracle (as it stands) on utterances b_ids of the workload, nthreads OpenMP threads."""
    import oracle
    pb = oracle_inputs(cfg, b_ids) if pb is None else pb
    z = pb["logits"].numpy()
    t0 = time.perf_counter()
    oracle.batch(z, pb["targets"], pb["logit_lens"], pb["target_lens"], cfg.blank, variant, grad=True,
                 nthreads=nthreads)
    return time.perf_counter() - t0


def n_chunks(B, cfg):
    """Utterance chunks of one call (<= 4 when the call has >= 2^24 elements, see rnnt_api.cu overlap_chunks)."""
    elems = B * cfg.Tmax * (cfg.Umax + 1) * cfg.V
    return min(B, 4) if (B >= 2 and elems >= (1 << 24)) else 1


def launches_per_step(mode, B, cfg):
    """Our kernels per step: K1/K2/K3 once per utterance chunk + the loss sum; viterbi = K1 + K4."""
    if mode == "viterbi":
        return 2
    if mode == "lattice":
        return 6 + 1  # K1, L2, L3, L4, L5, L6 + loss sum (plus one memset)
    return n_chunks(B, cfg) * (3 if mode == "loss_grad" else 2) + 1


def host_cores():
    return len(os.sched_getaffinity(0))


def host_avail_bytes():
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 64 << 30


def oracle_threads(cfg, want):
    """Threads (= utterances in flight) for the CPU oracle, bounded by cores and host memory (each utterance
    holds its fp32 logits and fp64 grads)."""
    per_utt = cfg.cells_per_utt * cfg.V * (4 + 8) * 1.1
    by_mem = int(0.5 * host_avail_bytes() // per_utt)
    return max(1, min(host_cores(), want, by_mem))


def run_reference(args):
    """--impl reference: the oracle on the host cores; each step = one utterance per thread."""
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return
    cfg = {**workloads.CONFIGS, **workloads.EXTRA_CONFIGS}[args.config]
    variant = args.variant or cfg.variant
    threads = oracle_threads(cfg, args.cpu_threads)
    import oracle
    oracle.build()
    b_ids = [i % cfg.B for i in range(threads)]
    pb = oracle_inputs(cfg, b_ids)                      # generated once, untimed
    for _ in range(min(args.warmup, 1)):               # the oracle has no warm-up state: one step pages it in
        oracle_sample(cfg, variant, threads, b_ids, pb)
    times = [oracle_sample(cfg, variant, threads, b_ids, pb) for _ in range(args.steps)]
    total = sum(times)
    value = len(b_ids) * args.steps / total
    sample = (f"{len(b_ids)} of the {cfg.B} utterances of {cfg.name} per step (one per thread), full "
              f"loss+grad per utterance, {args.steps} steps")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": ref_config(cfg, variant, args),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)


def ref_config(cfg, variant, args):
    """The GPU arm's config keys for the reference line (same workload, same batch per GPU)."""
    world = args.gpus
    gcfg = global_config(cfg, world, args.scaling)
    B = len(list(range(gcfg.B))[0::world]) if args.scaling == "strong" else cfg.B_per_gpu
    return {"workload": workload_desc(cfg, variant, args.dtype), "variant": variant, "B_per_gpu": B,
            "global_batch": gcfg.B, "parallelism": f"dp{world} (batch shards, NCCL all-reduce of the fp64 loss sum)",
            "l2": "n/a (host cores)", "grads": "out of place", "launch": "host (OpenMP, one utterance per thread)",
            "scaling": args.scaling}


# ------------------------------------------------------------------------------------------ GPU arm
def capture_steps(step, K, evs, world):
    """The K timed steps as one CUDA graph (and a second one carrying the per-kernel timing events).  At N > 1
    the NCCL all-reduce is captured with the kernels, so every N launches the same way."""
    graph, graph_ev = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        for i in range(K):
            step(None)
    with torch.cuda.graph(graph_ev):
        for i in range(K):
            step(evs[i] if evs is not None else None)
    graph.replay()  # one untimed replay each: a graph's first launch uploads it
    graph_ev.replay()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    return graph, graph_ev


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return subprocess.call(relaunch_cmd(sys.argv[1:], args.gpus, free_port()))

    import paper_2303_10384_b200 as rb
    from paper_2303_10384_b200 import dist as rdist

    rank, world, local = rdist.init(args.backend)
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    local = rdist.device_index(local, args.backend)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if args.mode in ("joint", "joint_grad"):
        return main_joint(args, rb, rdist, rank, world, local, dev)

    base = {**workloads.CONFIGS, **workloads.EXTRA_CONFIGS}[args.config]
    variant = args.variant or base.variant
    gcfg = global_config(base, world, args.scaling)
    b_ids = rdist.contiguous_shard(gcfg.B, rank, world)
    pb = workloads.problem(gcfg, b_ids=b_ids, device=dev)
    tdtype = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16}[args.dtype]
    if tdtype != torch.float32:
        pb["logits"] = pb["logits"].to(tdtype)
        torch.cuda.empty_cache()
    z = pb["logits"]
    esize = z.element_size()
    B, Tmax, Up1, V = z.shape
    Umax = Up1 - 1
    targets = torch.from_numpy(pb["targets"]).to(dev)
    T_b = torch.from_numpy(pb["logit_lens"]).to(dev)
    U_b = torch.from_numpy(pb["target_lens"]).to(dev)
    free, _ = torch.cuda.mem_get_info(dev)
    inplace = args.inplace or free < 1.05 * z.numel() * esize + (4 << 30)
    # out of place: logits stay fixed across steps; in place: later steps run on the previous step's grads
    # (same work -- the kernels' cost does not depend on the values)
    grads = z if inplace else torch.empty_like(z)
    losses = torch.empty(B, dtype=torch.float32, device=dev)
    loss_sum = torch.empty((), dtype=torch.float64, device=dev)
    workspace = torch.empty(rb.rnnt_workspace_bytes(B, Tmax, Umax), dtype=torch.uint8, device=dev)

    K, W = args.steps, args.warmup
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(K)]
    for row in evs:
        for e in row:
            e.record()  # create the CUDA handles
    torch.cuda.synchronize()

    dlat = None
    if args.mode == "lattice":
        from paper_2303_10384_b200 import lattice as rlat
        if args.lattice == "compose":
            from paper_2303_10384_b200 import compose as rcmp
            hl = rcmp.compose_lattices(pb["logit_lens"], pb["target_lens"], pb["targets"], gcfg.V, gcfg.blank, variant)
        else:
            hl = rlat.grid_lattices(pb["logit_lens"], pb["target_lens"], pb["targets"], gcfg.blank, variant)
        dlat = rb.lattice_to_device(hl, dev, Tmax, Umax)

    def step(events=None):
        if args.mode == "lattice":
            rb.rnnt_lattice_loss(z, dlat, T_b, U_b, grads=grads, losses=losses)
            rb.rnnt_loss_sum(losses, out=loss_sum)
            rdist.allreduce_loss_sum(loss_sum)
            return
        if args.mode == "viterbi":
            rb.rnnt_viterbi(z, targets, T_b, U_b, gcfg.blank, variant, workspace=workspace)
            return
        rb.rnnt_loss_timed(z, targets, T_b, U_b, gcfg.blank, variant, events=events,
                           grads=grads if args.mode == "loss_grad" else False, losses=losses, workspace=workspace)
        rb.rnnt_loss_sum(losses, out=loss_sum)
        rdist.allreduce_loss_sum(loss_sum)

    for _ in range(W):
        step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()

    graph = graph_ev = None
    if not args.eager and args.backend == "nccl" and args.mode in ("loss_grad", "loss"):
        # All K timed steps captured as one CUDA graph (replayed once below): every kernel of every step runs,
        # only the host launch overhead goes.  The C-ABI call forks its K2 chunks onto internal streams and
        # joins them back, so it is capturable (its internal streams were created by the warm-up calls); at
        # N > 1 the NCCL all-reduce of the loss sum is captured too (warmed up above).
        # Timing events inside a graph become external event nodes, which cost a few microseconds each, so
        # the per-kernel split comes from a second graph of the same K steps with the events, replayed right
        # after the timed one.
        graph, graph_ev = capture_steps(step, K, evs, world)

    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        start.record()
        if graph is not None:
            graph.replay()
        else:
            for i in range(K):
                step(evs[i])
        end.record()
        torch.cuda.synchronize()
    if graph_ev is not None:
        graph_ev.replay()
        torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    ms_local = start.elapsed_time(end)
    ms_total = rdist.max_over_ranks(ms_local, dev)
    ms_step = ms_total / K
    units = int(rdist.sum_over_ranks(B, dev))  # utterances all ranks processed per step
    value = units / (ms_step / 1e3)

    # per-kernel device durations inside the timed region (events: K1 start/end, K3 start/end, K2 start/end)
    def span(a, b_):
        return statistics.mean(r[a].elapsed_time(r[b_]) for r in evs)
    # (calls under 2^28 joint elements run each chunk's K3 on the chunk's stream right behind its K2: K3's span
    # then starts before K1's last chunk ends and overlaps it, and no K2 wait is exposed on the caller's stream)
    k_ms = {"k1_lse_gather": span(0, 1), "k2_alpha_beta": span(4, 5), "k3_grad": span(2, 3),
            "k2_exposed_wait": max(0.0, span(1, 2))}
    # per-step spread (median / p10 / p90): K1 start -> K3 end of each step, from the
    # event-carrying replay
    step_dist = None
    if args.mode == "loss_grad" and K >= 2:  # (loss mode has no event after the last chunk's K2)
        ends = 3
        per = sorted(r[0].elapsed_time(r[ends]) for r in evs)
        q = lambda f: per[min(len(per) - 1, int(round(f * (len(per) - 1))))]
        step_dist = {"p10": q(0.1), "p50": q(0.5), "p90": q(0.9), "n": len(per),
                     "span": "K1 start -> K3 end"}
    T_np, U_np = pb["logit_lens"], pb["target_lens"]
    valid_elems = int(sum(int(t) * (int(u) + 1) for t, u in zip(T_np, U_np))) * V
    all_elems = B * Tmax * Up1 * V
    k3_bytes = 2 * esize * valid_elems + esize * (all_elems - valid_elems)  # read+write valid, zero-write pad
    k1_bytes = esize * valid_elems
    peak, peak_src = measured_peaks()
    if args.mode != "loss_grad":  # no K3 (and, for viterbi, no per-kernel events): report K1 / the step
        k_ms["k3_grad"] = 0.0
        if args.mode in ("viterbi", "lattice"):
            k_ms = {f"step({args.mode})": ms_step}
    k3_gbs = k3_bytes / (k_ms["k3_grad"] / 1e3) / 1e9 if k_ms.get("k3_grad") else None
    k1_ms = k_ms.get("k1_lse_gather", ms_step)
    k1_gbs = k1_bytes / (k1_ms / 1e3) / 1e9
    peak, peak_src = measured_peaks()
    nch = n_chunks(B, gcfg)  # K1 / K3 launches per step (one per utterance chunk)
    if args.mode == "loss_grad":
        # per launch: the chunks' K3 launches run back to back on one stream, so the step's K3 bytes over the
        # events' K3 span = one launch's bytes over its mean duration
        traffic = ncu_traffic("k3_grad", args.config) if args.dtype == "f32" and world == 1 else None
        roof = {"bound": "hbm", "kernel": "k3_grad", "achieved": k3_gbs, "peak": peak, "unit": "GB/s",
                "frac": k3_gbs / peak, "traffic": traffic,
                "algorithmic_bytes_per_launch": k3_bytes / nch, "launches_per_step": nch,
                "algorithmic_bytes_per_step": k3_bytes, "peak_source": peak_src}
        if nch > 1 and B * Tmax * Up1 * V < (1 << 28):
            # small call (rnnt_api.cu): each chunk's K3 runs behind its K2 on the chunk's stream, overlapping the
            # later chunks' K1, so K3 has no span of its own -- report K1 + K3 bytes over K1-start -> K3-end
            both_ms = span(0, 3)
            gbs = (k1_bytes + k3_bytes) / (both_ms / 1e3) / 1e9
            roof = {"bound": "hbm", "kernel": "k1_lse_gather + k3_grad (overlapped, small call)", "achieved": gbs,
                    "peak": peak, "unit": "GB/s", "frac": gbs / peak, "traffic": None,
                    "algorithmic_bytes_per_launch": (k1_bytes + k3_bytes) / nch, "launches_per_step": nch,
                    "algorithmic_bytes_per_step": k1_bytes + k3_bytes, "peak_source": peak_src}
    else:
        nbytes = k1_bytes + (k3_bytes if args.mode == "lattice" else 0)  # lattice: the whole loss+grad step
        gbs = nbytes / ((k1_ms if args.mode == "loss" else ms_step) / 1e3) / 1e9
        per = nch if args.mode == "loss" else 1
        traffic = (ncu_traffic("k1_lse_gather", args.config) if args.mode == "loss" and args.dtype == "f32"
                   and world == 1 else None)
        roof = {"bound": "hbm", "kernel": "k1_lse_gather" if args.mode == "loss" else f"step ({args.mode})",
                "achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak,
                "traffic": traffic, "algorithmic_bytes_per_launch": nbytes / per,
                "launches_per_step": per, "algorithmic_bytes_per_step": nbytes, "peak_source": peak_src}

    # sanity: finite losses and the all-reduced sum
    loss_total = float(loss_sum.item())

    line = None
    if rank == 0:
        clk = clocks.summary()
        line = {
            "metric": METRIC if args.mode == "loss_grad" else f"utterances/s {args.mode} (not the BASELINE metric)",
            "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": ms_step, "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": args.dtype, "data": "synthetic",
            "config": {"workload": workload_desc(base, variant, args.dtype), "variant": variant, "B_per_gpu": B,
                       "global_batch": gcfg.B, "parallelism": f"dp{world} (batch shards, {args.backend.upper()} "
                       f"all-reduce of the fp64 loss sum)", "l2": f"inputs {z.numel() * esize / 1e9:.2f} GB/GPU > 126 MB L2: no flush",
                       "grads": "in place" if inplace else "out of place",
                       **({"lattice": args.lattice} if args.mode == "lattice" else {}),
                       "launch": (f"one CUDA graph of the {K} steps{' incl. the NCCL all-reduce' if world > 1 else ''} "
                                  f"(kernel split: a second graph of the same {K} steps with timing events, "
                                  f"replayed next)") if graph is not None else "eager",
                       "scaling": args.scaling},
            "roofline": roof,
            "kernels_ms": k_ms,
            "kernel_gbs": {"k1_lse_gather": k1_gbs, "k3_grad": k3_gbs},
            "note": None if args.dtype == "f32" else "16-bit storage run (SURVEY §8(f) NEXT-1); the BASELINE "
                    "metric itself is fp32",
            "kernel_frac_of_peak": {"k1_lse_gather": k1_gbs / peak, "k3_grad": k3_gbs and k3_gbs / peak},
            **({"step_frac_of_3pass_roofline": (3 * esize * valid_elems / (ms_step / 1e3) / 1e9) / peak,
                "step_frac_of_2pass_bound": (2 * esize * valid_elems / (ms_step / 1e3) / 1e9) / peak}
               if args.mode == "loss_grad" else {}),
            "step_ms_dist": step_dist,
            "clocks": clk,
            "gpu_launches": launches_per_step(args.mode, B, gcfg) * K,
            "loss_sum_last_step": loss_total,
        }

    # ---- end to end through the host-buffer C-ABI entry point (pinned host in/out, copies in the timed region)
    e2e = None
    if not args.no_e2e and args.mode != "loss_grad":
        e2e = {"value": None, "unit": UNIT, "reason": "the host-buffer entry point computes loss + grad"}
    elif not args.no_e2e and 2.2 * z.numel() * esize * int(os.environ.get("LOCAL_WORLD_SIZE", world)) > host_avail_bytes():
        e2e = {"value": None, "unit": UNIT, "reason": "pinned host copies of logits + grads exceed host RAM"}
    elif not args.no_e2e:
        zh = z.cpu().pin_memory()
        gh = torch.empty_like(zh).pin_memory()
        th = torch.from_numpy(pb["targets"]).contiguous().pin_memory()
        Th = torch.from_numpy(pb["logit_lens"]).pin_memory()
        Uh = torch.from_numpy(pb["target_lens"]).pin_memory()
        lh = torch.empty(B, dtype=torch.float32).pin_memory()
        if not inplace:
            del grads
        del z
        pb["logits"] = None
        torch.cuda.empty_cache()
        dbuf = torch.empty(rb.rnnt_host_buffer_bytes(B, Tmax, Umax, V, zh.dtype), dtype=torch.uint8, device=dev)
        for _ in range(1):
            rb.rnnt_loss_host(zh, th, Th, Uh, gcfg.blank, variant, losses_host=lh, grads_host=gh, device_buffer=dbuf)
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        e_start, e_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e_start.record()
        for _ in range(args.e2e_steps):
            rb.rnnt_loss_host(zh, th, Th, Uh, gcfg.blank, variant, losses_host=lh, grads_host=gh, device_buffer=dbuf)
        e_end.record()
        torch.cuda.synchronize()
        e_ms = rdist.max_over_ranks(e_start.elapsed_time(e_end), dev) / args.e2e_steps
        h2d = zh.numel() * esize + th.numel() * 4 + Th.numel() * 4 + Uh.numel() * 4
        d2h = gh.numel() * esize + lh.numel() * 4
        e2e = {"value": units / (e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": e_ms, "steps": args.e2e_steps,
               "api": f"rnnt_loss_host ({args.dtype} pinned host buffers; chunks of utterances through a 3-slot "
                      f"device ring, H2D / compute / D2H overlapped)"}
        del dbuf
    if rank == 0:
        line["e2e"] = e2e

    # ---- CPU baseline: the oracle as it stands, on the host cores, rank 0 at N=1 only
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = oracle_threads(base, args.cpu_threads)
        ids = [i % base.B_per_gpu for i in range(threads)]
        secs = oracle_sample(base, variant, threads, ids)
        secs1 = oracle_sample(base, variant, 1, ids[:1])  # the oracle on one core too
        line["cpu_baseline"] = {"value": len(ids) / secs, "unit": UNIT, "cores": threads, "kind": "oracle",
                                "sample": f"{len(ids)} utterances of {base.name} (one per OpenMP thread), full "
                                          f"double-precision loss+grad, {secs:.1f} s wall; single-core: 1 "
                                          f"utterance, {secs1:.2f} s",
                                "single_core_value": 1.0 / secs1,
                                "host_cores_available": host_cores()}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


# ------------------------------------------------------------------------------------------ fused joint (NEXT-4)
def main_joint(args, rb, rdist, rank, world, local, dev):
    """utterances/s of the fused joint network + loss forward (rnnt_joint_loss: K6 tcgen05 GEMM with the
    log-softmax / Populate epilogue, then K2), inputs = Encoder / Predictor embeddings of size H."""
    base = {**workloads.CONFIGS, **workloads.EXTRA_CONFIGS}[args.config]
    variant = args.variant or base.variant
    gcfg = global_config(base, world, args.scaling)
    b_ids = rdist.contiguous_shard(gcfg.B, rank, world)
    H = args.hidden
    T_np, U_np = workloads.lengths(gcfg)
    T_np, U_np = T_np[b_ids], U_np[b_ids]
    y_np = workloads.targets(gcfg, workloads.lengths(gcfg)[1], b_ids=b_ids)
    enc, pred, W, bias = workloads.joint_inputs(gcfg.B, gcfg.Tmax, gcfg.Umax, H, gcfg.V, seed=gcfg.logit_seed % 1000 + 1)
    enc, pred = enc[b_ids[0]:b_ids[-1] + 1].to(dev), pred[b_ids[0]:b_ids[-1] + 1].to(dev)
    W, bias = W.to(dev), bias.to(dev)
    B, Tmax, _ = enc.shape
    Umax, V = gcfg.Umax, gcfg.V
    targets = torch.from_numpy(y_np).to(dev)
    T_b = torch.from_numpy(T_np).to(dev)
    U_b = torch.from_numpy(U_np).to(dev)
    valid_rows = rb.joint_valid_rows(T_np, U_np, Tmax, Umax)  # host lengths: the GEMMs skip the padding
    losses = torch.empty(B, dtype=torch.float32, device=dev)
    loss_sum = torch.empty((), dtype=torch.float64, device=dev)
    grad = args.mode == "joint_grad"
    if grad:
        H_ = enc.shape[2]
        outs = (losses, torch.empty((B, Tmax, H_), device=dev), torch.empty((B, Umax + 1, H_), device=dev),
                torch.empty((V, H_), device=dev), torch.empty(V, device=dev))
        workspace = torch.empty(rb.library.rnnt_joint_grad_workspace_bytes(B, Tmax, Umax, H_, V), dtype=torch.uint8,
                                device=dev)
    else:
        workspace = torch.empty(rb.rnnt_workspace_bytes(B, Tmax, Umax), dtype=torch.uint8, device=dev)
    K, Wm = args.steps, args.warmup
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(K)]
    for row in evs:
        for e in row:
            e.record()
    torch.cuda.synchronize()

    def step(events=None):
        if grad:
            rb.rnnt_joint_loss_grad(enc, pred, W, bias, targets, T_b, U_b, gcfg.blank, variant, workspace=workspace,
                                    outputs=outs, valid_rows=valid_rows)
        else:
            rb.rnnt_joint_loss(enc, pred, W, bias, targets, T_b, U_b, gcfg.blank, variant, losses=losses,
                               workspace=workspace, events=events)
        rb.rnnt_loss_sum(losses, out=loss_sum)
        rdist.allreduce_loss_sum(loss_sum)

    for _ in range(Wm):
        step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    graph = graph_ev = None
    if not args.eager and args.backend == "nccl":
        graph, graph_ev = capture_steps(step, K, evs, world)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        start.record()
        if graph is not None:
            graph.replay()
        else:
            for i in range(K):
                step(evs[i])
        end.record()
        torch.cuda.synchronize()
    if graph_ev is not None:
        graph_ev.replay()
        torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    ms_step = rdist.max_over_ranks(start.elapsed_time(end), dev) / K
    units = int(rdist.sum_over_ranks(B, dev))
    value = units / (ms_step / 1e3)
    k6_ms = statistics.mean(r[0].elapsed_time(r[1]) for r in evs) if not grad else None
    k2_ms = statistics.mean(r[2].elapsed_time(r[3]) for r in evs) if not grad else None
    rows = int(sum(int(t) * (int(u) + 1) for t, u in zip(T_np, U_np)))  # K6 runs on the valid cells only
    flops = 2.0 * rows * V * H
    if grad:  # K6 forward + K6<grad> recompute + the two backward GEMMs, all over the valid cells (valid_rows)
        flops = 4 * 2.0 * rows * V * H
    tf = flops / ((ms_step if grad else k6_ms) / 1e3) / 1e12
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        mp = json.load(f)
    peak = float(mp["bf16_tflops_sustained"])
    loss_total = float(loss_sum.item())
    if rank != 0:
        if world > 1:
            torch.distributed.barrier()
            torch.distributed.destroy_process_group()
        return
    line = {
        "metric": ("utterances/s fused joint+loss training step (loss + d enc / d pred / dW / dbias; not the "
                   "BASELINE metric)") if grad else "utterances/s fused joint+loss forward (not the BASELINE metric)",
        "value": value, "unit": UNIT,
        "n_gpus": world, "steps": K, "warmup": Wm, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": f"{base.name} shapes through the joint: B={B}/GPU, Tmax={Tmax}, Umax={Umax}, "
                               f"V={V}, H={H} (enc/pred bf16, W [V,H] bf16, fp32 accumulate), "
                               f"{'RNN-T' if variant == 'rnnt' else 'W-RNNT ' + variant}",
                   "variant": variant, "B_per_gpu": B, "global_batch": gcfg.B, "H": H, "scaling": args.scaling,
                   "l2": "no flush: the joint's inputs (enc/pred/W, "
                         f"{(enc.numel() + pred.numel() + W.numel()) * 2 / 1e6:.0f} MB) are meant to be L2/HBM "
                         "resident; the [B,T,U+1,V] logits are never written",
                   "launch": ("one CUDA graph of the K steps" + ("" if grad else " (split from a second graph with events)"))
                             if graph is not None else "eager"},
        "roofline": {"bound": "tensor", "kernel": "step (joint_grad: 4 GEMM-sized passes)" if grad else "k6_joint_lse",
                     "achieved": tf, "peak": peak, "unit": "TFLOP/s",
                     "frac": tf / peak, "traffic": None if grad else ncu_traffic("k6_joint_lse", args.config + "_joint"), "algorithmic_flops_per_launch": flops,
                     "peak_source": "measured (MEASURED_PEAKS.json bf16_tflops_sustained: the kernel runs back "
                                    "to back inside the timed step)",
                     "frac_of_burst_peak": tf / float(mp["bf16_tflops"])},
        "kernels_ms": {"step": ms_step} if grad else {"k6_joint_lse": k6_ms, "k2_alpha_beta": k2_ms},
        "clocks": clocks.summary(),
        "gpu_launches": (9 if grad else 4) * K,  # rowmap, K6, K2, loss sum (+ K6<grad>, zero_tail, ones, K7 x2)
        "loss_sum_last_step": loss_total,
        "e2e": None,
    }
    if world == 1 and not args.no_cpu_baseline and not grad:
        from oracle import joint as oj
        ids = [0]
        t0 = time.perf_counter()
        oj.joint_loss(enc[:1].double().cpu().numpy(), pred[:1].double().cpu().numpy(), W.double().cpu().numpy(),
                      bias.double().cpu().numpy(), y_np[:1], T_np[:1], U_np[:1], gcfg.blank, variant)
        secs = time.perf_counter() - t0
        line["cpu_baseline"] = {"value": len(ids) / secs, "unit": UNIT, "cores": torch.get_num_threads(),
                                "kind": "oracle", "sample": f"1 utterance through oracle/joint.py (numpy fp64 "
                                f"joint + C loss oracle), {secs:.1f} s wall"}
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main() or 0)

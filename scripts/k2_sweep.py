"""Time K1/K2/K3 on the c3 workload for several K2 cells-per-lane settings (RNNT_K2_CELLS)."""
import os, sys, statistics, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads
import paper_2303_10384_b200 as rb

cfg = workloads.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
variants = sys.argv[2].split(",") if len(sys.argv) > 2 else ["rnnt"]
pb = workloads.problem(cfg, device="cuda")
z = pb["logits"]; B, Tmax, Up1, V = z.shape
tg = torch.from_numpy(pb["targets"]).cuda(); T = torch.from_numpy(pb["logit_lens"]).cuda(); U = torch.from_numpy(pb["target_lens"]).cuda()
grads = torch.empty_like(z); losses = torch.empty(B, device="cuda")
ws = torch.empty(rb.rnnt_workspace_bytes(B, Tmax, Up1 - 1), dtype=torch.uint8, device="cuda")
out = {}
for variant in variants:
    for cells in ("1", "2", "4", "8"):
        os.environ["RNNT_K2_CELLS"] = cells
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(20)]
        for r in evs:
            for e in r: e.record()
        for i in range(25):
            rb.rnnt_loss_timed(z, tg, T, U, cfg.blank, variant, events=evs[i % 20], grads=grads, losses=losses, workspace=ws)
        torch.cuda.synchronize()
        k = [statistics.median(r[a].elapsed_time(r[b]) for r in evs) for a, b in ((0, 1), (4, 5), (2, 3), (1, 2), (0, 3))]
        out[f"{variant}_C{cells}"] = {"k1_ms": k[0], "k2_ms": k[1], "k3_ms": k[2], "wait_ms": k[3], "total_ms": k[4],
                                      "loss0": float(losses[0])}
print(json.dumps(out, indent=1))

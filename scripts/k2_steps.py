"""K2 cost per wavefront step vs U (B=1 -> sequential path, one CTA per direction)."""
import os, sys, statistics, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads
import paper_2303_10384_b200 as rb
res = {}
for variant in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["rnnt"]):
    for U in (15, 31, 63, 100, 127, 200, 400):
        T, V = 500, 64
        cfg = workloads.Config("k2", B=1, Tmax=T, Umax=U, V=V, logit_seed=3)
        pb = workloads.problem(cfg, device="cuda")
        z = pb["logits"]
        tg = torch.from_numpy(pb["targets"]).cuda(); Tb = torch.from_numpy(pb["logit_lens"]).cuda(); Ub = torch.from_numpy(pb["target_lens"]).cuda()
        ws = torch.empty(rb.rnnt_workspace_bytes(1, T, U), dtype=torch.uint8, device="cuda")
        losses = torch.empty(1, device="cuda")
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(20)]
        for r in evs:
            for e in r: e.record()
        for i in range(30):
            rb.rnnt_loss_timed(z, tg, Tb, Ub, 0, variant, events=evs[i % 20], grads=False, losses=losses, workspace=ws)
        torch.cuda.synchronize()
        ms = statistics.median(r[4].elapsed_time(r[5]) for r in evs)
        res[f"{variant}_U{U}"] = {"k2_us": ms * 1e3, "ns_per_step": ms * 1e6 / (T + U)}
print(json.dumps(res, indent=1))

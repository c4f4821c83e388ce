"""Summarise an ncu --set full report of one bench step (K1/K2/K3, possibly split in utterance chunks)
into profiles/<tag>_ncu_full.txt and the per-step DRAM traffic table profiles/ncu_traffic.json."""
import csv, io, json, subprocess, sys, os, collections

rep, tag, cfg = sys.argv[1], sys.argv[2], (sys.argv[3] if len(sys.argv) > 3 else "c3")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
ix = {h: i for i, h in enumerate(hdr)}
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes.sum.per_second",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct"]
scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "Tbyte": 1e12}
agg = collections.OrderedDict()
out = [f"# ncu --set full --clock-control none ({tag}); one bench step of {cfg}; kernels launched per utterance chunk",
       f"# report: {os.path.basename(rep)}"]
for r in rows[2:]:
    name = r[ix["Kernel Name"]].split("(")[0].split("::")[-1]  # strip the argument list first
    fam = name.split("<")[0]
    out.append(f"\n[{name}]  grid={r[ix['launch__grid_size']]} block={r[ix['launch__block_size']]}")
    for k in keys:
        if k in ix:
            out.append(f"  {k:62s} {r[ix[k]]:>16s} {units[ix[k]]}")
    a = agg.setdefault(fam, {"launches": 0, "dram_read": 0.0, "dram_write": 0.0, "duration_ms_cold": 0.0})
    a["launches"] += 1
    a["dram_read"] += float(r[ix["dram__bytes_read.sum"]]) * scale[units[ix["dram__bytes_read.sum"]]]
    a["dram_write"] += float(r[ix["dram__bytes_write.sum"]]) * scale[units[ix["dram__bytes_write.sum"]]]
    d = float(r[ix["gpu__time_duration.sum"]])
    a["duration_ms_cold"] += d if units[ix["gpu__time_duration.sum"]] == "ms" else d / 1e3
out.append("\n# per-step totals (all chunk launches of one step)")
for fam, a in agg.items():
    a["dram_bytes_per_launch"] = a["dram_read"] + a["dram_write"]
    a["note"] = "per step: sum over the step's chunk launches"
    a["source"] = f"profiles/{tag}_ncu_full.txt"
    out.append(f"  {fam:16s} launches={a['launches']} dram={a['dram_bytes_per_launch']/1e9:.4f} GB "
               f"cold_ms={a['duration_ms_cold']:.4f} -> {a['dram_bytes_per_launch']/1e9/a['duration_ms_cold']:.3f} TB/s")
open(f"profiles/{tag}_ncu_full.txt", "w").write("\n".join(out) + "\n")
tpath = "profiles/ncu_traffic.json"
t = json.load(open(tpath)) if os.path.exists(tpath) else {}
t[cfg] = agg
json.dump(t, open(tpath, "w"), indent=1)
print("\n".join(out[-len(agg) - 1:]))

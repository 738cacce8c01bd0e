"""Summarise a round's ncu outputs (gpurun_out/<R>_*) into profiles/<R>_summary.md + traffic.json."""
import csv, json, os, re, statistics, subprocess, sys
R = sys.argv[1] if len(sys.argv) > 1 else "r1"
G = "gpurun_out"
out = []
# ---- launch list
rows = list(csv.reader(open(f"{G}/{R}_launches.csv")))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi, ii = h.index("Kernel Name"), h.index("Metric Value"), h.index("ID")
launches = [(int(r[ii]), re.sub(r"\(.*", "", r[ki]).replace("void ", "").replace("q4::", ""), float(r[vi]))
            for r in rows[hi + 1:] if len(r) > vi and r[vi]]
# the eager forward: first quantize after the weight prep, then 24 x 5 kernels
names = [n for _, n, _ in launches]
start = next(i for i in range(len(names)) if names[i].startswith("quantize_rows") and i + 1 < len(names)
             and names[i + 1].startswith("w4a4_tc_kernel"))
fwd = launches[start:start + 1 + 24 * 5]
roles = ["qkv_gemm_f16", "attention_q4", "attn_out_gemm_resln_q4", "ffn1_gemm_gelu_q4", "ffn2_gemm_resln_q4"]
per = {r: [] for r in roles}
for j, (_, n, t) in enumerate(fwd[1:]):
    per[roles[j % 5]].append(t)
tot = sum(t for _, _, t in fwd)
out.append(f"# {R} profile summary\n")
out.append(f"ncu launch list (`gpu__time_duration.sum`, `--clock-control none`, serialised, cold) of "
           f"`bench.py --steps 2 --warmup 1 --no-extras --no-cpu-baseline --no-e2e` (file `{R}_launches.csv`).\n"
           f"Eager forward of the bench workload (BERT-large, 24 layers, M = 32768): "
           f"{len(fwd)} launches, {tot/1e6:.2f} ms total.\n")
out.append("| kernel | launches | median us | share of forward |\n|---|---|---|---|")
out.append(f"| quantize_rows (layer-0 input) | 1 | {fwd[0][2]/1e3:.1f} | {fwd[0][2]/tot:.3f} |")
for r in roles:
    out.append(f"| {r} | {len(per[r])} | {statistics.median(per[r])/1e3:.1f} | {sum(per[r])/tot:.3f} |")
# ---- full captures
rep = f"{G}/{R}_layer.ncu-rep"
traffic = {}
if os.path.exists(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    hh, data = rr[0], rr[2:]
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed.avg.per_cycle_active", "launch__registers_per_thread",
            "launch__shared_mem_per_block_dynamic", "launch__grid_size", "launch__block_size",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
            "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]
    units = rr[1]
    out.append(f"\n`ncu --set full` of one layer's five kernels (`{R}_layer.ncu-rep`, M = 32768):\n")
    out.append("| kernel | " + " | ".join(k.split(".")[0].replace("__", ".") + f" [{units[hh.index(k)]}]" for k in keys if k in hh) + " |")
    out.append("|---" * (1 + sum(k in hh for k in keys)) + "|")
    for j, d in enumerate(data):
        name = re.sub(r"\(.*", "", d[hh.index("Kernel Name")]).replace("void ", "").replace("q4::", "")
        out.append(f"| {name} ({roles[j] if j < 5 else ''}) | " + " | ".join(d[hh.index(k)] for k in keys if k in hh) + " |")
        if j < 5:
            rd = float(d[hh.index("dram__bytes_read.sum")]); wr = float(d[hh.index("dram__bytes_write.sum")])
            mult = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1}[units[hh.index("dram__bytes_read.sum")]]
            traffic[f"large:{roles[j]}:M32768"] = (rd + wr) * mult
open(f"profiles/{R}_summary.md", "w").write("\n".join(out) + "\n")
if traffic:
    json.dump(traffic, open("profiles/traffic.json", "w"), indent=1)
print("\n".join(out))

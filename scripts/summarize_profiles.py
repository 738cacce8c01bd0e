"""Summarise a round's ncu outputs into profiles/<R>/summary.md + traffic.json.

Step 1 (only when the scratch captures exist): copy gpurun_out/<R>_launches.csv and export
`ncu -i gpurun_out/<R>_layer.ncu-rep --page raw --csv` into profiles/<R>/ (committed).
Step 2: every number of the summary is computed from those committed CSVs, so
`python scripts/summarize_profiles.py <R>` regenerates it from the repository alone."""
import csv, json, os, re, shutil, statistics, subprocess, sys
R = sys.argv[1] if len(sys.argv) > 1 else "r2"
G = "gpurun_out"
P = f"profiles/{R}"
os.makedirs(P, exist_ok=True)
if os.path.exists(f"{G}/{R}_launches.csv"):
    shutil.copy(f"{G}/{R}_launches.csv", f"{P}/launches.csv")
if os.path.exists(f"{G}/{R}_layer.ncu-rep"):
    raw = subprocess.run(["ncu", "-i", f"{G}/{R}_layer.ncu-rep", "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    open(f"{P}/layer_raw.csv", "w").write(raw)
out = []
# ---- launch list
rows = list(csv.reader(open(f"{P}/launches.csv")))
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
           f"`bench.py --steps 2 --warmup 1 --no-extras --no-cpu-baseline --no-e2e` (file `{P}/launches.csv`).\n"
           f"Eager forward of the bench workload (BERT-large, 24 layers, M = 32768): "
           f"{len(fwd)} launches, {tot/1e6:.2f} ms total.\n")
out.append("| kernel | launches | median us | share of forward |\n|---|---|---|---|")
out.append(f"| quantize_rows (layer-0 input) | 1 | {fwd[0][2]/1e3:.1f} | {fwd[0][2]/tot:.3f} |")
for r in roles:
    out.append(f"| {r} | {len(per[r])} | {statistics.median(per[r])/1e3:.1f} | {sum(per[r])/tot:.3f} |")
# ---- roofline fractions of the serialised launch times (algorithmic work: bench.py)
sys.path.insert(0, os.getcwd())
import bench  # noqa: E402
pk = bench.peaks()
M, h, f, H = 32768, 1024, 4096, 16
work = {"qkv_gemm_f16": bench.gemm_work(M, 3 * h, h, "f16"), "attention_q4": bench.attention_work(256, 128, H),
        "attn_out_gemm_resln_q4": bench.gemm_work(M, h, h, "resln_q4"),
        "ffn1_gemm_gelu_q4": bench.gemm_work(M, f, h, "gelu_q4"), "ffn2_gemm_resln_q4": bench.gemm_work(M, h, f, "resln_q4")}
out.append(f"\nRoofline of the serialised (cold, ncu) launch times; peaks from MEASURED_PEAKS.json: INT8 = 2 x bf16 "
           f"({pk['int8_tops']:.0f} TOPS sustained, {pk['int8_tops_burst']:.0f} burst), HBM {pk['hbm_gbs']:.0f} GB/s. "
           f"A kernel inside the long step is held to the sustained figure.\n")
out.append("| kernel | median us | TOPS | GB/s | bound | frac (sustained) | frac (burst) |\n|---|---|---|---|---|---|---|")
ridge = pk["int8_tops"] * 1e12 / (pk["hbm_gbs"] * 1e9)
for r in roles:
    t = statistics.median(per[r]) * 1e-9
    ops, by = work[r]
    tops, gbs = ops / t / 1e12, by / t / 1e9
    if "gemm" in r and ops / by > ridge:
        out.append(f"| {r} | {t*1e6:.1f} | {tops:.0f} | {gbs:.0f} | tensor | {tops/pk['int8_tops']:.2f} | {tops/pk['int8_tops_burst']:.2f} |")
    else:
        out.append(f"| {r} | {t*1e6:.1f} | {tops:.0f} | {gbs:.0f} | hbm | {gbs/pk['hbm_gbs']:.2f} | {gbs/pk['hbm_gbs']:.2f} |")
# ---- full captures
traffic = {}
if os.path.exists(f"{P}/layer_raw.csv"):
    rr = list(csv.reader(open(f"{P}/layer_raw.csv")))
    hh, data = rr[0], rr[2:]
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed.avg.per_cycle_active", "launch__registers_per_thread",
            "launch__shared_mem_per_block_dynamic", "launch__grid_size", "launch__block_size",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
            "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]
    units = rr[1]
    out.append(f"\n`ncu --set full` of one layer's five kernels (raw export `{P}/layer_raw.csv`, M = 32768):\n")
    out.append("| kernel | " + " | ".join(k.split(".")[0].replace("__", ".") + f" [{units[hh.index(k)]}]" for k in keys if k in hh) + " |")
    out.append("|---" * (1 + sum(k in hh for k in keys)) + "|")
    for j, d in enumerate(data):
        name = re.sub(r"\(.*", "", d[hh.index("Kernel Name")]).replace("void ", "").replace("q4::", "")
        out.append(f"| {name} ({roles[j] if j < 5 else ''}) | " + " | ".join(d[hh.index(k)] for k in keys if k in hh) + " |")
        if j < 5:
            rd = float(d[hh.index("dram__bytes_read.sum")]); wr = float(d[hh.index("dram__bytes_write.sum")])
            mult = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1}[units[hh.index("dram__bytes_read.sum")]]
            traffic[f"large:{roles[j]}:M32768"] = (rd + wr) * mult
# ---- latency config: BERT-base 12 layers, batch 1 (warm launch list, scripts/probe_latency.py)
if os.path.exists(f"{G}/{R}_bs1_launches.csv"):
    shutil.copy(f"{G}/{R}_bs1_launches.csv", f"{P}/bs1_launches.csv")
if os.path.exists(f"{P}/bs1_launches.csv"):
    rows = list(csv.reader(open(f"{P}/bs1_launches.csv")))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, gi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Grid Size")
    ls = [(re.sub(r"\(.*", "", r[ki]).replace("void ", "").replace("q4::", ""), float(r[vi]), r[gi])
          for r in rows[hi + 1:] if len(r) > vi and r[vi]]
    last = ls[-61:]  # the last eager forward: quantize + 12 x 5 kernels
    roles1 = ["qkv_gemm_f16", "attention_q4", "attn_out_gemm_resln_q4", "ffn1_gemm_gelu_q4", "ffn2_gemm_resln_q4"]
    per1 = {r: [] for r in roles1}
    grid1 = {}
    for j, (n, t, g) in enumerate(last[1:]):
        per1[roles1[j % 5]].append(t)
        grid1[roles1[j % 5]] = g
    tot1 = sum(t for _, t, _ in last)
    out.append(f"\nLatency config (BERT-base, 12 layers, batch 1, seq 128): ncu launch list with "
               f"`--cache-control none` (warm L2, serialised: no PDL overlap) of `scripts/probe_latency.py 12 1` "
               f"(file `{P}/bs1_launches.csv`); {len(last)} launches, {tot1/1e3:.1f} us summed.\n")
    out.append("| kernel | grid | median us |\n|---|---|---|")
    out.append(f"| quantize_rows (layer-0 input) | {last[0][2]} | {last[0][1]/1e3:.2f} |")
    for r in roles1:
        out.append(f"| {r} | {grid1[r]} | {statistics.median(per1[r])/1e3:.2f} |")
open(f"{P}/summary.md", "w").write("\n".join(out) + "\n")
if traffic:
    json.dump(traffic, open(f"{P}/traffic.json", "w"), indent=1)
    json.dump(traffic, open("profiles/traffic.json", "w"), indent=1)  # what bench.py quotes
print("\n".join(out))

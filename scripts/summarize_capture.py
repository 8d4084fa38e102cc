"""Turn one `scripts/round_capture.sh` output directory into the tracked
summaries under profiles/ (bench lines, launch list + per-kernel shares,
ncu key metrics of the generation and tensor-core fitness kernels, the
fitness sweep as CSV, phase timing).

Usage: python scripts/summarize_capture.py gpurun_out/r01c r01
"""
import csv
import json
import shutil
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

src, pre = Path(sys.argv[1]), sys.argv[2]
dst = Path(__file__).resolve().parents[1] / "profiles"
US = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}
PEAK = json.load(open(Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json"))["hbm_gbs"]

for a, b in (("bench.json", "bench.json"), ("bench_ref.json", "bench_ref.json"), ("launches.csv", "bench_launches.csv"),
             ("phase.jsonl", "phase_timing.jsonl")):
    if (src / a).exists():
        shutil.copy(src / a, dst / f"{pre}_{b}")

# launch list -> per-kernel totals
rows = [r for r in csv.reader(open(src / "launches.csv")) if len(r) > 10] if (src / "launches.csv").exists() else []
hdr = rows[0] if rows else ["Kernel Name", "Metric Name", "Metric Value"]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
agg = defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    if r[mi] == "gpu__time_duration.sum":
        v = float(r[vi].replace(",", ""))
        unit = r[hdr.index("Metric Unit")]
        us = v * US[unit]
        name = r[ki].split("(")[0][:60]
        agg[name][0] += 1
        agg[name][1] += us
tot = sum(v[1] for v in agg.values())
with open(dst / f"{pre}_bench_launches_summary.csv" if rows else "/dev/null", "w") as f:
    f.write("kernel,launches,total_us,share\n")
    for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        f.write(f"{k},{n},{us:.1f},{us / tot:.3f}\n")


def raw(rep):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(out.splitlines()))
    return {h: (u, v) for h, u, v in zip(rr[0], rr[1], rr[2])}


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__pipe_tensor_subpipe_imma_cycles_active.avg",
        "sm__cycles_elapsed.avg", "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"]


def to_bytes(u, v):
    x = float(v.replace(",", ""))
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


for rep, m in (("fit_tc48.ncu-rep", 48), ("fit_tc64.ncu-rep", 64)):
    if not (src / rep).exists():
        continue
    d = raw(src / rep)
    met = {k: list(d[k]) for k in KEYS if k in d}
    n = 1_000_000
    t_us = float(d["gpu__time_duration.sum"][1].replace(",", "")) * US[d["gpu__time_duration.sum"][0]]
    rd = to_bytes(*d["dram__bytes_read.sum"])
    wr = to_bytes(*d["dram__bytes_write.sum"])
    alg = n * (m * m + 8)
    json.dump({"kernel": f"{'k_fit_i8_tc2' if pre >= 'r02' else 'k_fit_i8_tc'}<{m},F2> (tcgen05.mma.kind::i8 column Gram, "
                         f"{n:,} int8 {m}x{m} matrices)",
               "source": f"ncu --set full --clock-control none, `python scripts/prof_tc.py {m} {n}`; {src}/{rep}",
               "metrics": met, "algorithmic_bytes": alg, "dram_bytes": rd + wr, "traffic_over_algorithmic": (rd + wr) / alg,
               "evals_per_s_under_ncu": n / (t_us * 1e-6), "achieved_GBps": alg / (t_us * 1e-6) / 1e9,
               "frac_of_hbm": alg / (t_us * 1e-6) / 1e9 / PEAK},
              open(dst / f"{pre}_fit_tc{m}_ncu.json", "w"), indent=1)

if (src / "k_run.ncu-rep").exists():
    d = raw(src / "k_run.ncu-rep")
    json.dump({"kernel": "k_run_v3<20,F2,5,0> (one generation inside bench.py, L2 flushed before it)",
               "source": f"ncu --set full -k regex:k_run_v3 -s 30 -c 1 python bench.py --steps 40 --warmup 3 --no-sweep --no-cpu; {src}/k_run.ncu-rep",
               "metrics": {k: list(d[k]) for k in KEYS if k in d},
               "algorithmic_bytes_per_launch": 5_440_000},
              open(dst / f"{pre}_k_run_traffic.json", "w"), indent=1)

# fitness sweep -> CSV
popc = json.loads((Path(__file__).resolve().parents[1] / "profiles" / "r02_peaks.json").read_text())["popc_per_s"]
with open(dst / f"{pre}_fitness_sweep.csv", "w") as f:
    f.write("m,n,kernel,path,variant,evals_per_s,GBps,hbm_ceiling_evals,popc_ceiling_evals,frac_of_hbm\n")
    for line in open(src / "fitness_sweep.jsonl"):
        r = json.loads(line)
        if "kernel" not in r:
            continue
        m = r["m"]
        W = (m + 31) // 32
        if r["kernel"] == "fitness_i8":
            b = m * m + 8 * (1 if r["variant"] != "all" else 4)
        else:
            b = 4 * m * W + 8
        hbm = PEAK * 1e9 / b
        pc = popc / (m * (m - 1) / 2 * W)
        f.write(f"{m},{r['n']},{r['kernel']},{r.get('path', 'popc')},{r['variant']},{r['evals_per_s']:.4g},"
                f"{r['GBps']:.0f},{hbm:.4g},{pc:.4g},{r['evals_per_s'] / hbm:.3f}\n")
print("ok")

"""Per-source-line totals from `ncu -i X --page source --csv --print-source cuda,sass`."""
import csv
import subprocess
import sys
from collections import defaultdict


def main(rep, top=40, kernel_idx=None):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    agg = defaultdict(lambda: [0.0, 0.0, ""])
    file = func = None
    hdr = None
    nfunc = 0
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            file = r[1].split("/")[-1]
            continue
        if r[0] == "Function Name":
            func = r[1]
            nfunc += 1
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 8 or not r[0].isdigit():
            continue
        if kernel_idx is not None and nfunc != kernel_idx:
            continue
        try:
            s = float(r[4] or 0)
            n = float(r[7] or 0)
        except ValueError:
            continue
        key = (func[:40] if func else "?", file, int(r[0]) if r[0].isdigit() else -1)
        agg[key][0] += s
        agg[key][1] += n
        agg[key][2] = r[1][:100]
    tot_s = sum(v[0] for v in agg.values()) or 1
    tot_n = sum(v[1] for v in agg.values()) or 1
    print(f"total samples {tot_s:.0f}, warp instrs {tot_n:.0f}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{k[1]}:{k[2]:<5} {100*v[0]/tot_s:5.1f}%smp {100*v[1]/tot_n:5.1f}%ins  {v[2]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40, int(sys.argv[3]) if len(sys.argv) > 3 else None)

"""Summarise an ncu --page source --print-source sass CSV: hottest SASS by
stall samples and by executed instructions (one kernel per CSV block)."""
import csv
import sys


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    blocks, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1], "rows": []}
            blocks.append(cur)
        elif r and r[0] == "Address":
            cur["hdr"] = r
        elif cur is not None and "hdr" in cur and len(r) == len(cur["hdr"]):
            cur["rows"].append(dict(zip(cur["hdr"], r)))
    for b in blocks[:1] if len(sys.argv) < 4 else blocks:
        rs = b["rows"]
        def f(r, k):
            try:
                return float(r.get(k, 0) or 0)
            except ValueError:
                return 0.0
        tot_s = sum(f(r, "Warp Stall Sampling (All Samples)") for r in rs)
        tot_i = sum(f(r, "Instructions Executed") for r in rs)
        print(f"== {b['name']}  samples={tot_s:.0f} warp_instrs={tot_i:.0f}")
        for key in ("Warp Stall Sampling (All Samples)", "Instructions Executed"):
            print(f"-- top by {key}")
            for r in sorted(rs, key=lambda r: -f(r, key))[:top]:
                print(f"{r['Address']:>8} {f(r,'Warp Stall Sampling (All Samples)'):7.0f} {f(r,'Instructions Executed'):10.0f}  {r['Source'][:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)

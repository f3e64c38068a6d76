"""Per-instruction issue counts of one kernel from an ncu source-page CSV (--page source --print-source sass):
prints the hottest address ranges (basic blocks by executed count) and totals.  Usage:
python tools/sass_hist.py source.csv[.gz] [min_share]"""
import csv
import gzip
import io
import sys

path = sys.argv[1]
mins = float(sys.argv[2]) if len(sys.argv) > 2 else 0.002
raw = gzip.open(path, "rt").read() if path.endswith(".gz") else open(path).read()
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[1]
ia, isrc, iex, ith, ism = (hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed"),
                           hdr.index("Avg. Threads Executed"), hdr.index("Warp Stall Sampling (All Samples)"))
ins = []
for r in rows[2:]:
    if len(r) <= iex or not r[ia].startswith("0x"):
        continue
    ins.append((int(r[ia], 16), r[isrc].strip(), int(r[iex] or 0), float(r[ith] or 0), int(r[ism] or 0)))
tot = sum(x[2] for x in ins)
tsm = sum(x[4] for x in ins) or 1
base = ins[0][0]
print(f"total warp instructions {tot:.4e}, stall samples {tsm}")
# blocks: maximal runs of consecutive instructions with the same executed count
blocks = []
for a, s, e, th, sm in ins:
    if blocks and blocks[-1]["e"] == e:
        blocks[-1]["n"] += 1
        blocks[-1]["sm"] += sm
        blocks[-1]["last"] = a
        blocks[-1]["src"].append(s)
    else:
        blocks.append({"first": a, "last": a, "e": e, "n": 1, "th": th, "sm": sm, "src": [s]})
for b in blocks:
    share = b["e"] * b["n"] / tot
    if share >= mins:
        print(f"{b['first'] - base:#07x}-{b['last'] - base:#07x} n={b['n']:3d} exec={b['e']:.3e} share={share:6.3f} "
              f"thr={b['th']:4.1f} stall={b['sm'] / tsm:6.3f} | {' ; '.join(x.split(',')[0] for x in b['src'][:4])}")

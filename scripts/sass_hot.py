"""Summarise an ncu SASS source page (CSV): shared wavefronts/conflicts per instruction and per
contiguous region.   python scripts/sass_hot.py src_sass.csv[.gz]"""
import csv, gzip, sys
f = sys.argv[1]
op = gzip.open if f.endswith(".gz") else open
rows = list(csv.reader(op(f, "rt")))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
def g(r, k):
    try: return float(r[ix[k]])
    except Exception: return 0.0
tot_w = sum(g(r, "L1 Wavefronts Shared") for r in data)
tot_i = sum(g(r, "L1 Wavefronts Shared Ideal") for r in data)
tot_s = sum(g(r, "Warp Stall Sampling (All Samples)") for r in data)
tot_e = sum(g(r, "Instructions Executed") for r in data)
print(f"shared wavefronts {tot_w:.4g} ideal {tot_i:.4g} stall samples {tot_s:.4g} warp-instr {tot_e:.4g}")
# regions: split at BAR.SYNC
reg, cur = [], {"start": 0, "w": 0, "wi": 0, "s": 0, "e": 0, "g": 0, "fp": 0, "n": 0}
for k, r in enumerate(data):
    src = r[ix["Source"]].strip()
    cur["w"] += g(r, "L1 Wavefronts Shared"); cur["wi"] += g(r, "L1 Wavefronts Shared Ideal")
    cur["s"] += g(r, "Warp Stall Sampling (All Samples)"); cur["e"] += g(r, "Instructions Executed")
    cur["g"] += g(r, "L2 Theoretical Sectors Global")
    if "DFMA" in src or "DMUL" in src or "DADD" in src: cur["fp"] += g(r, "Instructions Executed")
    cur["n"] += 1
    if "BAR.SYNC" in src or k == len(data) - 1:
        cur["end"] = k
        reg.append(cur)
        cur = {"start": k + 1, "w": 0, "wi": 0, "s": 0, "e": 0, "g": 0, "fp": 0, "n": 0}
print("region  [start-end]   shared_wf  (ideal)   stall%   instr%  fp64instr  sectorsG")
for q in reg:
    print(f"[{q['start']:5d}-{q['end']:5d}] {q['w']/1e6:9.2f}M ({q['wi']/1e6:7.2f}M) {100*q['s']/tot_s:6.1f} {100*q['e']/tot_e:7.1f} {q['fp']/1e6:9.2f}M {q['g']/1e6:8.2f}M")

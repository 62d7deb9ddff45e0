"""Aggregate an ncu --csv launch list (gpu__time_duration, dram bytes) by kernel name over the
last `n` launches: python scripts/kernel_table.py launches.csv [n_last]"""
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
data = rows[1:]
# one row per (launch, metric)
by = collections.OrderedDict()
for r in data:
    try:
        key = (r[ix["ID"]], r[ix["Kernel Name"]])
    except Exception:
        continue
    by.setdefault(key, {})[r[ix["Metric Name"]]] = (float(r[ix["Metric Value"]].replace(",", "")), r[ix["Metric Unit"]])
items = list(by.items())
if len(sys.argv) > 2 and not sys.argv[2].isdigit():   # from the last launch whose name contains it
    k = max(i for i, ((_, nm), _) in enumerate(items) if sys.argv[2] in nm)
    items = items[k:]
else:
    n = int(sys.argv[2]) if len(sys.argv) > 2 else len(items)
    items = items[-n:]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
tot = 0.0
for (lid, name), m in items:
    t, u = m.get("gpu__time_duration.sum", (0, "ns"))
    t = t * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "nsecond": 1e-9, "ms": 1e-3, "msecond": 1e-3}.get(u, 1e-9)
    b = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        v, uu = m.get(k, (0, "byte"))
        b += v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(uu, 1)
    nm = name.split("(")[0].replace("void ", "")[:70]
    a = agg[nm]
    a[0] += 1; a[1] += t; a[2] += b
    tot += t
print(f"{'kernel':70s} {'n':>4s} {'ms':>9s} {'%':>6s} {'GB':>8s} {'GB/s':>8s}")
for nm, (c, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{nm:70s} {c:4d} {t*1e3:9.3f} {100*t/tot:6.1f} {b/1e9:8.2f} {b/t/1e9 if t else 0:8.0f}")
print(f"total {tot*1e3:.3f} ms over {len(items)} launches")

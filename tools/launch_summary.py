"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) of bench.py:
the kernels of ONE decomposition (from its k_iota to its last k_post_col)."""
import collections
import csv
import gzip
import sys

path = sys.argv[1]
op = gzip.open if path.endswith(".gz") else open
rows = [r for r in csv.reader(op(path, "rt")) if len(r) > 5]
hdr, data = rows[0], rows[1:]
ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
seq = []
for r in data:
    try:
        seq.append((r[ik].split("(")[0].replace("void ", "").strip(), float(r[iv].replace(",", ""))))
    except ValueError:
        pass
iota = [i for i, (k, _) in enumerate(seq) if k.endswith("k_iota")]
start = iota[-1]
ends = [i for i, (k, _) in enumerate(seq) if k.endswith("k_post_col") and i > start]
end = ends[-1] + 1
seg = seq[start:end]
d = collections.defaultdict(list)
for k, v in seg:
    d[k].append(v)
tot = sum(v for _, v in seg)
print(f"one decomposition: launches {len(seg)}, serialized sum {tot / 1e6:.3f} ms")
print(f"{'kernel':34s} {'launches':>8s} {'ms':>9s} {'share':>6s}")
for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:34s} {len(v):8d} {sum(v) / 1e6:9.3f} {100 * sum(v) / tot:5.1f}%")

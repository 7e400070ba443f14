"""Print kernel / metric / value rows of an ncu --csv --metrics log."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]
k, m, v = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
for r in rows[h + 1:]:
    print(r[k][:48], r[m], r[v])

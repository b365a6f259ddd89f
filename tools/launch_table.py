"""Print the per-launch table of an `ncu --metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum --csv` log (kernel, grid, us, MB)."""
import collections
import csv
import sys


def rows(path):
    lines = [l for l in open(path) if not l.startswith("==")]
    r = list(csv.reader(lines))
    h = r[0]
    k, m, v, i, g = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID", "Grid Size"))
    d = collections.OrderedDict()
    for x in r[1:]:
        e = d.setdefault(x[i], {"kernel": x[k].split("(")[0].split("::")[-1], "grid": x[g]})
        e[x[m]] = float(x[v].replace(",", ""))
    return list(d.values())


if __name__ == "__main__":
    last = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    for e in rows(sys.argv[1])[-last:]:
        t = e.get("gpu__time_duration.sum", 0) / 1e3
        mb = (e.get("dram__bytes_read.sum", 0) + e.get("dram__bytes_write.sum", 0)) / 1e6
        print(f"{e['kernel'][:34]:34s} {e['grid']:>14s} {t:9.1f} us {mb:9.1f} MB {mb / t if t else 0:6.2f} TB/s")

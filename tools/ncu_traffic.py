"""Per-launch DRAM traffic of the hot kernels from ncu raw CSV pages.

    python tools/ncu_traffic.py out.json <ne>:raw_<ne>.csv[.gz] ...

Writes {"bytes_per_launch": {kernel: {ne: dram read + write bytes}}, "time_us":
...} averaged over the launches of each kernel (tools/kernel_probe.py runs each
twice), keyed by the short template name bench.py looks up (ncu_traffic()).
"""
import csv
import gzip
import io
import json
import re
import sys


def short(name):
    base = name.split("(")[0] if "(" not in name.split("<")[0] else name
    m = re.search(r"(\w+_kernel)<([^>]*)>", name)
    if not m:
        return name.split("(")[0].split()[-1]
    args = [re.sub(r"\((bool|int)\)", "", a).strip() for a in m.group(2).split(",")]
    if m.group(1) == "mgs2_kernel":
        args = args[:4]
    return f"{m.group(1)}<{','.join(args)}>"


def scale(v, unit):
    f = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6,
         "ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    return float(v) * f[unit]


def main():
    out, items = sys.argv[1], sys.argv[2:]
    res = {"bytes_per_launch": {}, "time_us": {}, "source": {}}
    for it in items:
        ne, path = it.split(":", 1)
        op = gzip.open if path.endswith(".gz") else open
        with op(path, "rt") as fh:
            rows = list(csv.reader(fh))
        hdr, units, body = rows[0], rows[1], rows[2:]
        ix = {h: i for i, h in enumerate(hdr)}
        acc = {}
        for r in body:
            k = short(r[ix["Kernel Name"]])
            rd = scale(r[ix["dram__bytes_read.sum"]], units[ix["dram__bytes_read.sum"]])
            wr = scale(r[ix["dram__bytes_write.sum"]], units[ix["dram__bytes_write.sum"]])
            t = scale(r[ix["gpu__time_duration.sum"]], units[ix["gpu__time_duration.sum"]])
            a = acc.setdefault(k, [0.0, 0.0, 0])
            a[0] += rd + wr
            a[1] += t
            a[2] += 1
        for k, (b, t, n) in acc.items():
            res["bytes_per_launch"].setdefault(k, {})[ne] = round(b / n)
            res["time_us"].setdefault(k, {})[ne] = round(t / n, 2)
        res["source"][ne] = path.split("/")[-1]
    with open(out, "w") as fh:
        json.dump(res, fh, indent=1, sort_keys=True)
    print(json.dumps(res["bytes_per_launch"], indent=1))


if __name__ == "__main__":
    main()

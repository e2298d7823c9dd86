"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes):
per-kernel-family launch count, mean duration and mean DRAM bytes, and the
per-pass list of the first sort.  Usage: launch_summary.py launches.csv [--json]"""
import collections
import csv
import json
import sys


OURS = ("tile_sort_kernel", "merge_kernel", "mergepath_", "merge_bitonic_kernel",
        "merge_partition_kernel", "split64", "join64")


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            name = d["Kernel Name"]
            if "b200" not in name and not any(x in name for x in OURS):
                continue  # (ncu prints names without the namespace unless asked to)
            e = data.setdefault(d["ID"], {"name": d["Kernel Name"]})
            e[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    return list(data.values())


def family(name):
    if "tile_sort" in name:
        return "tile_sort"
    if "mergepath_merge" in name:
        return "mergepath_merge"  # the merge-path sort variant's phase tiles
    if "mergepath_partition" in name:
        return "mergepath_partition"
    if "merge_bitonic_kernel" in name:
        return "merge_path"  # the merge-path tiles (multi-GPU / host entry)
    if "merge_kernel" in name or "cluster_merge" in name:
        return "merge"
    return name.split("(")[0].split()[-1]


def summarise(path):
    ls = load(path)
    fam = collections.OrderedDict()
    for d in ls:
        f = fam.setdefault(family(d["name"]), {"launches": 0, "us": 0.0, "dram": 0.0})
        f["launches"] += 1
        f["us"] += d["gpu__time_duration.sum"] / 1e3
        f["dram"] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
    for f in fam.values():
        f["mean_us"] = f["us"] / f["launches"]
        f["mean_dram_bytes"] = f["dram"] / f["launches"]
    # first sort: from the first tile-sort launch to the launch before the next one
    first = []
    for d in ls:
        if "tile_sort_kernel" in d["name"] and first:
            break
        if "tile_sort_kernel" in d["name"] or first:
            first.append(d)
    return ls, fam, first


if __name__ == "__main__":
    ls, fam, first = summarise(sys.argv[1])
    if "--json" in sys.argv:  # per-family DRAM bytes per launch of the FIRST sort
        out = collections.OrderedDict()
        for d in first:
            f = out.setdefault(family(d["name"]), [0, 0.0])
            f[0] += 1
            f[1] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
        print(json.dumps({k: round(v[1] / v[0]) for k, v in out.items()}))
        sys.exit(0)
    print(f"# {sys.argv[1]}: {len(ls)} launches of this library's kernels")
    print("# (ncu replay: serialised, cold-cache, no PDL overlap -- shares, not absolutes)")
    for k, v in fam.items():
        print(f"{k:12s} launches {v['launches']:5d}  mean {v['mean_us']:9.2f} us  "
              f"mean DRAM {v['mean_dram_bytes'] / 1e6:10.3f} MB/launch")
    tot = sum(d["gpu__time_duration.sum"] for d in first) / 1e3
    print(f"# first sort: {len(first)} passes, {tot:.1f} us serialised")
    for d in first:
        t = d["gpu__time_duration.sum"] / 1e3
        b = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
        print("%-62s %9.1f us %8.1f MB %7.0f GB/s" % (
            d["name"].replace("void b200::", "").replace("(b200::PassParams)", "")[:62], t,
            b / 1e6, b / (t * 1e-6) / 1e9 if t else 0))

"""Summarise ncu --set full reports (per launch: time, DRAM bytes, throughput,
occupancy, top stall reasons) into one JSON file for profiles/.

    python tools/ncu_summary.py out.json rep1.ncu-rep [rep2.ncu-rep ...]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "TPC.TriageCompute.sm__pipe_fp64_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"]


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True)
    data = list(csv.reader(io.StringIO(out.stdout)))
    return data[0], data[1], data[2:]


def main():
    dst, reps = sys.argv[1], sys.argv[2:]
    launches = []
    for rep in reps:
        hdr, units, body = rows(rep)
        idx = {h: i for i, h in enumerate(hdr)}
        stall = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_")
                 and h.endswith("_per_issue_active.ratio")]
        for r in body:
            item = {"report": rep.split("/")[-1], "kernel": r[idx["Kernel Name"]].split("(")[0]}
            for k in KEYS:
                if k in idx:
                    item[f"{k} [{units[idx[k]]}]"] = r[idx[k]]
            st = []
            for h in stall:
                try:
                    st.append((float(r[idx[h]]), h[len("smsp__average_warps_issue_stalled_"):-len(
                        "_per_issue_active.ratio")]))
                except ValueError:
                    pass
            item["top_stalls_per_issue"] = [[n, round(v, 3)] for v, n in sorted(st, reverse=True)[:4]]
            launches.append(item)
    with open(dst, "w") as fh:
        json.dump({"launches": launches}, fh, indent=1)
    for it in launches:
        print(it["kernel"][:48], {k.split(".")[0].split("__")[-1]: v for k, v in it.items()
                                   if "fp64" in k or "dram__bytes" in k or "duration" in k})


if __name__ == "__main__":
    main()

"""Summaries committed under profiles/ from gpurun_out/ ncu outputs.

    python profiles/summarize_ncu.py launches <launches.csv> <out.txt> <title>
    python profiles/summarize_ncu.py full <report.ncu-rep> <out.json> <config> <algorithmic_bytes> [<traffic.json>]
"""
import collections
import csv
import json
import subprocess
import sys

CONV = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}


def launches(path, out, title):
    rows = list(csv.reader(open(path)))
    hdr, agg = None, collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] != "gpu__time_duration.sum":
                continue
            name = d["Kernel Name"].split("(")[0].split("::")[-1]
            agg.setdefault(name, []).append(float(d["Metric Value"].replace(",", "")) * CONV[d["Metric Unit"]])
    tot = sum(sum(v) for v in agg.values())
    lines = [f"{title}: {sum(len(v) for v in agg.values())} launches"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append("%-22s launches=%3d mean_us=%10.1f share=%5.1f%%" % (k, len(v), sum(v) / len(v),
                                                                         100 * sum(v) / tot))
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def full(rep, out, config, alg_bytes, traffic_out=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "lts__throughput.avg.pct_of_peak_sustained_elapsed", "launch__shared_mem_per_block_dynamic",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
            "sm__warps_active.avg.pct_of_peak_sustained_active"]
    o = {}
    for w in want:
        if w in hdr:
            i = hdr.index(w)
            o[w] = vals[i]
            o[w + ".unit"] = units[i]
    st = [(hdr[i].replace("smsp__pcsamp_warps_issue_stalled_", ""), vals[i]) for i in range(len(hdr))
          if hdr[i].startswith("smsp__pcsamp_warps_issue_stalled") and not hdr[i].endswith("not_issued")]
    st = sorted([(float(v.replace(",", "")), k) for k, v in st if v.replace(",", "").replace(".", "").isdigit()],
                reverse=True)[:8]
    o["top_stalls"] = [[k, int(v)] for v, k in st]
    mul = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}
    traffic = (float(o["dram__bytes_read.sum"].replace(",", "")) * mul[o["dram__bytes_read.sum.unit"]] +
               float(o["dram__bytes_write.sum"].replace(",", "")) * mul[o["dram__bytes_write.sum.unit"]])
    o["algorithmic_bytes_per_launch"] = int(alg_bytes)
    o["dram_traffic_per_launch"] = int(traffic)
    o["note"] = (f"k_scan_tc, {config}, one launch, ncu --set full --clock-control none "
                 "(replayed: the duration is cold-cache/serialised, compare shares not absolutes)")
    json.dump(o, open(out, "w"), indent=1)
    json.dump({"config": config, "kernel": "k_scan_tc", "dram_bytes_per_launch": int(traffic),
               "source": out + " (ncu --set full, one launch)"},
              open(traffic_out or out.replace("r1_ncu_k_scan_tc_", "ncu_traffic_"), "w"), indent=1)
    print(json.dumps(o, indent=1)[:900])


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(*sys.argv[2:5])
    else:
        full(*sys.argv[2:7])

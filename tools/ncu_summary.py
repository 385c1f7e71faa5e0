"""Summarise ncu outputs into profiles/.

    python tools/ncu_summary.py launches gpurun_out/launches.csv  > profiles/rNN_launches.txt
    python tools/ncu_summary.py full gpurun_out/fmha.ncu-rep       > profiles/rNN_fmha_ncu.txt
"""
import collections
import csv
import io
import re
import subprocess
import sys

NCU = "/usr/local/cuda/bin/ncu"


def short(name):
    name = re.sub(r"\(.*", "", name)
    return name[:90]


def launches(path):
    text = open(path).read()
    i = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[i:])))
    agg = collections.defaultdict(lambda: [0, 0.0])
    total = 0.0
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        ns = v * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(unit, 1)
        k = short(r["Kernel Name"])
        agg[k][0] += 1
        agg[k][1] += ns
        total += ns
    print(f"# ncu launch list ({sum(a[0] for a in agg.values())} launches, {total / 1e6:.2f} ms serialised, cold-cache)")
    print(f"{'share':>7} {'total_ms':>10} {'count':>6} {'avg_us':>10}  kernel")
    for k, (n, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{100 * ns / total:6.2f}% {ns / 1e6:10.3f} {n:6d} {ns / n / 1e3:10.1f}  {k}")


WANT = ["gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__cycles_elapsed.avg.per_second", "smsp__inst_executed.sum",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_xu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum"]


def full(path):
    out = subprocess.run([NCU, "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if not rows:
        print("no data")
        return
    hdr = rows[0]
    units = rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    for r in rows[2:]:
        print(f"## {short(r[idx['Kernel Name']])}  (id {r[idx['ID']]})")
        for m in WANT:
            if m in idx:
                print(f"  {m:70s} {r[idx[m]]:>18} {units[idx[m]]}")
        # all tensor / pipe metrics present
        for h, i in idx.items():
            if ("pipe_tensor" in h or "pipe_tc" in h) and h not in WANT and "pct" in h:
                print(f"  {h:70s} {r[i]:>18} {units[i]}")
        print()


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])

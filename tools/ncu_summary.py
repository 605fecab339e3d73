"""Summaries of ncu output for profiles/: a launch list (CSV from
`ncu --metrics gpu__time_duration.sum --csv --log-file`) -> per-kernel share
of GPU time; a `--set full` report -> the key metrics as JSON.

    python tools/ncu_summary.py launches LIST.csv > profiles/..._summary.txt
    python tools/ncu_summary.py report REP.ncu-rep > profiles/..._metrics.json
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "lts__t_bytes.sum.per_second", "l1tex__t_bytes.sum.per_second",
        "lts__t_sectors_srcunit_tex_op_read.sum", "smsp__inst_executed.sum",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed"]


def launches(path):
    rows = list(csv.reader(open(path)))
    head = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[head]
    k, v, u = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[head + 1:]:
        if len(r) <= v or not r[v]:
            continue
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
                 "nsecond": 1e-6}.get(r[u], 1.0)
        name = r[k].split("(")[0]
        tot[name] += float(r[v].replace(",", "")) * scale
        cnt[name] += 1
    all_ms = sum(tot.values())
    print("launches   total ms   share  kernel")
    for name in sorted(tot, key=tot.get, reverse=True):
        print(f"{cnt[name]:8d} {tot[name]:10.3f} {100 * tot[name] / all_ms:6.1f}%  {name}")


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    res = {}
    for key in KEYS:
        if key in hdr:
            i = hdr.index(key)
            res[key] = [vals[i], units[i]]
    # per-pipe utilisation (which execution pipe, if any, is the limiter)
    for i, key in enumerate(hdr):
        if (key.startswith("sm__inst_executed_pipe_") and key.endswith(".avg.pct_of_peak_sustained_active")) \
                or key in ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
                           "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed"):
            res[key] = [vals[i], units[i]]
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    {"launches": launches, "report": report}[sys.argv[1]](sys.argv[2])

#!/usr/bin/env python
"""Summaries of ncu output for profiles/ (B200_PROFILING.md recipe).

    python scripts/ncu_summary.py launches <launch-list.csv>          # --metrics gpu__time_duration.sum
    python scripts/ncu_summary.py full <raw.csv> [<source.csv>]        # ncu -i rep --page raw --csv

`launches`: per kernel name the launch count, total and per-launch time and share (cold-cache,
serialised: compare shares, not absolutes).  `full`: per launch the duration, DRAM bytes, DRAM
utilisation, issue and XU utilisation, warp occupancy, registers and the top stall reasons; with
a source-page csv also the SASS lines with the most stall samples.
"""

import collections
import csv
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(list)
    for r in rows[hdr + 1:]:
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        ms = v / 1e6 if unit == "ns" else v / 1e3 if unit in ("us", "usecond") else v
        name = r[ki].split("(")[0]
        agg[name].append(ms)
    tot = sum(sum(v) for v in agg.values())
    print("# kernel | launches | total ms | share | ms/launch")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print("%-44s %6d %11.3f %7.2f%% %10.4f" % (k[:44], len(v), sum(v), 100 * sum(v) / tot, sum(v) / len(v)))
    print("total %.3f ms over %d launches" % (tot, sum(len(v) for v in agg.values())))


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size"]


def full(raw, src=None):
    rows = list(csv.reader(open(raw)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        print(d.get("Kernel Name", "?").split("(")[0])
        for m in METRICS:
            if m in d:
                print("   %-58s %-10s %s" % (m, units[hdr.index(m)], d[m]))
        st = []
        for k in hdr:
            if "issue_stalled" in k and k.endswith("per_issue_active.ratio") and d.get(k) not in ("", "n/a", None):
                st.append((float(d[k]), k.replace("smsp__average_warps_issue_stalled_", "")
                           .replace("_per_issue_active.ratio", "")))
        print("   stalls (warps per issue):", ", ".join("%s %.2f" % (n, v) for v, n in sorted(st, reverse=True)[:8]))
    if src:
        s = list(csv.reader(open(src)))
        h = s[1] if s[0] and s[0][0] != "Address" else s[0]
        start = 2 if h is s[1] else 1
        ia, isrc, iss = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
        data = []
        for r in s[start:]:
            try:
                data.append((int(r[iss]), r[ia], r[isrc][:90]))
            except (ValueError, IndexError):
                pass
        tot = sum(x[0] for x in data) or 1
        print("   top SASS by stall samples (%d total):" % tot)
        for x in sorted(data, reverse=True)[:12]:
            print("    %6d %5.1f%%  %s" % (x[0], 100.0 * x[0] / tot, x[2]))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        full(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)

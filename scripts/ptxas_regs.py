#!/usr/bin/env python
"""Summarise `ptxas -v` output (from `python -m paper_2404_08970_b200._build -v`): one line per kernel
with registers, spills and static shared memory.  Usage: ptxas_regs.py LOG [name-regex]"""
import re
import subprocess
import sys

log = open(sys.argv[1]).read().splitlines()
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
name = None
spill = ""
for line in log:
    m = re.search(r"Compiling entry function '([^']+)'", line)
    if m:
        name = m.group(1)
        spill = ""
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and name:
        spill = "" if m.group(1) == "0" and m.group(2) == "0" else " SPILL %s/%s" % (m.group(1), m.group(2))
    m = re.search(r"Used (\d+) registers.*?(\d+) bytes smem", line)
    if m and name:
        dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
        dem = re.sub(r"\(.*", "", dem)
        if pat is None or pat.search(dem):
            print("%4s regs %6s B smem%s  %s" % (m.group(1), m.group(2), spill, dem))
        name = None

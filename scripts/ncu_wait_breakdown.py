#!/usr/bin/env python
"""Where the pair kernel's warps wait: sums ncu's warp-state samples (`--page source --csv
--print-source sass` of a `--set full` capture) over each mbarrier try-wait loop, by barrier
(offset in the kernel's barrier block), so the MMA issuer's waits for operand data (full
barriers), for a free accumulator (tempty) and the producer's waits for a free stage (empty) can
be compared.  usage: python scripts/ncu_wait_breakdown.py REPORT.ncu-rep"""
import csv
import io
import re
import subprocess
import sys

NAMES = {0x30000: "full: the MMA issuer waits for a stage's operands", 0x30030: "empty: the producer waits for a free stage",
         0x30060: "tfull: epilogue warps wait for an accumulator", 0x30070: "tempty: the MMA issuer waits for the epilogue",
         0x30080: "rfull: consumers wait for the next item", 0x300a0: "rempty: the scheduler waits for a ring slot"}


def main():
    txt = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, data = rows[1], rows[2:]
    isrc, iall = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
    s = lambda r: int(r[iall]) if r[iall].isdigit() else 0  # noqa: E731
    by = {}
    for k, r in enumerate(data):
        m = re.search(r"TRYWAIT P(\d), \[(R\d+)\+(URZ|UR\d+)\+0x(300[0-9a-f]{2})\]", r[isrc])
        if not m:
            continue
        p, off = m.group(1), int(m.group(4), 16) & ~0xF if int(m.group(4), 16) >= 0x30060 else None
        off = int(m.group(4), 16)
        base = max(b for b in NAMES if b <= off)
        tot = s(r) + (s(data[k - 1]) if "YIELD" in data[k - 1][isrc] else 0)
        for j in range(k + 1, min(k + 5, len(data))):
            if "BRA" in data[j][isrc] and ("@!P" + p) in data[j][isrc]:
                tot += s(data[j])
        by[base] = by.get(base, 0) + tot
    issue = sum(s(data[j]) for k, r in enumerate(data) if "UTCHMMA" in r[isrc] for j in range(k, k + 1))
    print(f"total warp samples {sum(s(r) for r in data)}")
    for b in sorted(by):
        print(f"  {by[b]:8d}  {NAMES[b]}")
    print(f"  {issue:8d}  on the UTCHMMA instructions themselves")


if __name__ == "__main__":
    main()

"""Summarise gpurun_out/ ncu artefacts into committed files under profiles/.

  python scripts/summarize_profiles.py r01

Writes profiles/<round>_launches.csv (per-launch times of one bench step),
profiles/<round>_ncu_summary.md and profiles/ncu_summary.json (per-class DRAM
bytes per launch, read by bench.py for the roofline `traffic` field).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

METRICS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum",
    "lts__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread", "launch__grid_size",
    "launch__cluster_dim_x", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "derived__lts__lts2xbar_bytes.sum.per_second", "l1tex__m_xbar2l1tex_read_bytes.sum",
    "lts__t_sectors_srcunit_ltcfabric.sum", "l1tex__data_bank_reads.avg.pct_of_peak_sustained_elapsed",
]


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (vals[i], units[i]) for i, h in enumerate(hdr)}


def to_bytes(v, u):
    v = float(v.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)


def main(rnd):
    os.makedirs(PROF, exist_ok=True)
    lines = [f"# ncu summary, round {rnd}", "",
             "Captured with `scripts/profile_round.sh` on one B200 (`ncu --set full --clock-control none`),",
             "first timed step of `bench.py` (Qwen2.5-0.5B head: N=8192, D=896, V=151936, 40% ignored).",
             "ncu replays serialise and run cold: compare shares and counters, not absolute times.", ""]
    summary = {"round": rnd, "per_class_dram_bytes_per_launch": {}, "kernels": {}}
    for name, cls in (("prof_fwd", "fwd_logits_lse"), ("prof_bwd", "bwd")):
        rep = os.path.join(OUT, name + ".ncu-rep")
        if not os.path.exists(rep):
            continue
        r = raw(rep)
        lines.append(f"## {cls} (`{r.get('Kernel Name', ('?', ''))[0][:60]}`)")
        lines.append("")
        lines.append("| metric | value | unit |")
        lines.append("|---|---|---|")
        for m in METRICS:
            if m in r:
                lines.append(f"| {m} | {r[m][0]} | {r[m][1]} |")
        lines.append("")
        rd = to_bytes(*r["dram__bytes_read.sum"])
        wr = to_bytes(*r["dram__bytes_write.sum"])
        summary["per_class_dram_bytes_per_launch"][cls] = rd + wr
        summary["kernels"][cls] = {m: r[m][0] + " " + r[m][1] for m in METRICS if m in r}
    # launch list
    lpath = os.path.join(OUT, "launches.csv")
    if os.path.exists(lpath):
        rows = list(csv.reader(open(lpath)))
        hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
        hdr = rows[hi]
        ki, mi, vi, ui, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
        per = {}
        for r in rows[hi + 1:]:
            per.setdefault((int(r[ii]), r[ki]), {})[r[mi]] = (r[vi], r[ui])
        with open(os.path.join(PROF, f"{rnd}_launches.csv"), "w") as f:
            f.write("id,kernel,time_ns,dram_read_bytes,dram_write_bytes\n")
            for (i, k), m in sorted(per.items()):
                t = m.get("gpu__time_duration.sum", ("0", "ns"))
                tn = float(t[0].replace(",", "")) * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(t[1], 1)
                rd = to_bytes(*m.get("dram__bytes_read.sum", ("0", "byte")))
                wr = to_bytes(*m.get("dram__bytes_write.sum", ("0", "byte")))
                f.write(f"{i},\"{k.split('(')[0]}\",{tn:.0f},{rd:.0f},{wr:.0f}\n")
        # share of one (the last) bench step: our kernels only
        ours = [(i, k, m) for (i, k), m in sorted(per.items()) if "cce::" in k or "pairk::" in k]
        lines.append("## launch list (last bench step, our kernels, ncu serialised)")
        lines.append("")
        lines.append("| kernel | time (us) | DRAM read (MB) | DRAM write (MB) |")
        lines.append("|---|---|---|---|")
        starts = [n for n, (i, k, m) in enumerate(ours) if "k_label_scan" in k]
        step = ours[starts[-1]:] if starts else ours
        tot = 0.0
        for i, k, m in step:
            t = m.get("gpu__time_duration.sum", ("0", "ns"))
            tn = float(t[0].replace(",", "")) * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(t[1], 1)
            tot += tn
            lines.append(f"| {k.split('(')[0].replace('void ', '')} | {tn / 1e3:.1f} | {to_bytes(*m.get('dram__bytes_read.sum', ('0', 'byte'))) / 1e6:.1f} | "
                         f"{to_bytes(*m.get('dram__bytes_write.sum', ('0', 'byte'))) / 1e6:.1f} |")
        lines.append(f"| total | {tot / 1e3:.1f} | | |")
        lines.append("")
    open(os.path.join(PROF, f"{rnd}_ncu_summary.md"), "w").write("\n".join(lines) + "\n")
    json.dump(summary, open(os.path.join(PROF, "ncu_summary.json"), "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")

#!/usr/bin/env python
"""Summarize ncu reports (.ncu-rep, from `ncu --set full`) into a short text table per kernel.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [...] > profiles/rNN_ncu_<name>.txt
    python tools/ncu_summary.py --traffic KEY REGEX rep   # print dram bytes/launch of kernels matching REGEX
"""
import csv
import io
import re
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 sector hit rate %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 (LTS) throughput %"),
    ("lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed", "L2 atomic input active %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "L1TEX throughput %"),
    ("l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed", "L1->XBAR request cycles %"),
    ("l1tex__m_xbar2l1tex_read_bytes.sum", "XBAR->L1 read bytes"),
    ("l1tex__m_l1tex2xbar_write_bytes.sum", "L1->XBAR write bytes"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active % (achieved occupancy)"),
    ("smsp__inst_executed.sum", "warp instructions executed"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def summarize(rep):
    h, u, data = raw(rep)
    lines = [f"# {rep}"]
    for v in data:
        name = v[h.index("Kernel Name")]
        lines.append(f"\n## {name}")
        for key, label in METRICS:
            if key in h:
                i = h.index(key)
                lines.append(f"  {label:40s} {v[i]:>18s} {u[i]}")
        stalls = []
        for i, n in enumerate(h):
            m = re.match(r"smsp__pcsamp_warps_issue_stalled_(\w+)$", n)
            if m and not n.endswith("not_issued"):
                try:
                    stalls.append((float(v[i]), m.group(1)))
                except ValueError:
                    pass
        tot = sum(s for s, _ in stalls) or 1.0
        top = ", ".join(f"{nm} {100 * s / tot:.0f}%" for s, nm in sorted(stalls, reverse=True)[:6])
        lines.append(f"  {'stall samples (top)':40s} {top}")
    return "\n".join(lines)


def traffic(rep, regex):
    h, u, data = raw(rep)
    vals = []
    for v in data:
        if re.search(regex, v[h.index("Kernel Name")]):
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            r = float(v[h.index("dram__bytes_read.sum")]) * scale[u[h.index("dram__bytes_read.sum")]]
            w = float(v[h.index("dram__bytes_write.sum")]) * scale[u[h.index("dram__bytes_write.sum")]]
            vals.append(r + w)
    return sum(vals) / len(vals) if vals else None


if __name__ == "__main__":
    if sys.argv[1] == "--traffic":
        print(traffic(sys.argv[4], sys.argv[3]))
    else:
        for rep in sys.argv[1:]:
            print(summarize(rep))

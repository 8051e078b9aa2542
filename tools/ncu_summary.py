"""Summarise an ncu report (raw page) into the metrics the roofline uses."""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % of peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("lts__t_bytes.sum", "L2 bytes"),
]


def summarise(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    lines = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        lines.append(f"### {d.get('Kernel Name', '?')[:140]}")
        for k, name in KEYS:
            if k in d:
                lines.append(f"- {name}: {d[k]} {u.get(k, '')}".rstrip())
        stalls = []
        for h, v in d.items():
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    stalls.append((float(v.replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        tot = sum(s for s, _ in stalls) or 1.0
        lines.append("- top stall reasons (pc sampling): " +
                     ", ".join(f"{n} {100 * s / tot:.0f}%" for s, n in stalls[:5]))
    return "\n".join(lines)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(f"## {p}\n")
        print(summarise(p))
        print()

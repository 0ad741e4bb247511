"""Summarise ncu outputs into profiles/ text files.

  python tools/ncu_summary.py launches <launches.csv> <out.txt>   # launch list -> per-kernel shares
  python tools/ncu_summary.py full <report.ncu-rep> <out.txt>     # key metrics of a --set full capture
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

FULL_METRICS = [
    "gpu__time_duration.sum",
    "launch__grid_size",
    "launch__block_size",
    "launch__registers_per_thread",
    "launch__shared_mem_per_block_static",
    "launch__shared_mem_per_block_dynamic",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_op_tcgen05_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_sleeping_per_issue_active.ratio",
]


_UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1.0, "usecond": 1e3, "msecond": 1e6}


def launches(path, out):
    """Per-kernel launch counts, device time (ns -> ms) and, when captured, DRAM read/write bytes."""
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr_i]
    ik, iv, im, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name"), h.index("Metric Unit")
    tot = defaultdict(float)
    rd = defaultdict(float)
    wr = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[hdr_i + 1:]:
        if len(r) <= iv:
            continue
        name = r[ik].split("(")[0].replace("void ", "").replace("cmsvd::", "")
        v = float(r[iv].replace(",", "")) * _UNIT.get(r[iu], 1.0)
        if r[im] == "gpu__time_duration.sum":
            tot[name] += v
            cnt[name] += 1
        elif r[im] == "dram__bytes_read.sum":
            rd[name] += v
        elif r[im] == "dram__bytes_write.sum":
            wr[name] += v
    s = sum(tot.values())
    dram = bool(rd)
    lines = [f"{'kernel':40s} {'launches':>8s} {'total_ms':>10s} {'share':>7s}" +
             (f" {'dram_rd_GB':>10s} {'dram_wr_GB':>10s}" if dram else "")]
    for k in sorted(tot, key=lambda k: -tot[k]):
        lines.append(f"{k[:40]:40s} {cnt[k]:8d} {tot[k] / 1e6:10.3f} {100 * tot[k] / s:6.2f}%" +
                     (f" {rd[k] / 1e9:10.3f} {wr[k] / 1e9:10.3f}" if dram else ""))
    lines.append(f"{'total':40s} {sum(cnt.values()):8d} {s / 1e6:10.3f}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def full(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    lines = []
    for r in rows[2:]:
        lines.append("Kernel: " + r[h.index("Kernel Name")])
        for m in FULL_METRICS:
            if m in h:
                lines.append(f"  {m:80s} {r[h.index(m)]:>16s} {rows[1][h.index(m)]}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2], sys.argv[3])

"""Summarise an .ncu-rep (raw page) into the metrics we track; used to write profiles/."""
import csv, io, subprocess, sys

WANT = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA cycles %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("l1tex__t_bytes.sum", "L1 bytes"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__warps_active.avg.per_cycle_active", "warps active / SM"),
    ("launch__registers_per_thread", "registers"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def summarize(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    return "\n".join(_one(hdr, units, vals) for vals in rows[2:])


def _one(hdr, units, vals):
    idx = {h: i for i, h in enumerate(hdr)}
    out = [f"kernel: {vals[idx['Kernel Name']][:100]}"]
    for key, label in WANT:
        if key in idx:
            out.append(f"  {label:22s} {vals[idx[key]]} {units[idx[key]]}")
    stalls = [(h.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(vals[i].replace(",", "") or 0))
              for h, i in idx.items() if h.startswith("smsp__pcsamp_warps_issue_stalled_")
              and not h.endswith("not_issued")]
    tot = sum(v for _, v in stalls) or 1.0
    out.append("  top stall reasons (pc sampling): " + ", ".join(
        f"{n} {100 * v / tot:.0f}%" for n, v in sorted(stalls, key=lambda x: -x[1])[:6]))
    return "\n".join(out)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(summarize(p))

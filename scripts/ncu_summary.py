"""Summarise an ncu --set full report (ncu -i rep --page raw --csv) into the metrics the
roofline and DESIGN.md cite: duration, SM clock, tensor-pipe activity, DRAM bytes and
throughput, L2 hit rate / throughput, L2->SM traffic, registers, achieved occupancy, and
the top warp-stall reasons.

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/<name>.txt
"""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__m_xbar2l1tex_read_bytes.sum", "l1tex__m_xbar2l1tex_read_bytes.sum.per_second",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
]


def main(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        print(f"# {r[hdr.index('Kernel Name')][:110]}")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"  {k:70s} {r[i]:>18s} {units[i]}")
        stalls = [(h, r[i]) for i, h in enumerate(hdr)
                  if h.startswith("smsp__average_warp_latency_issue_stalled") and h.endswith(".ratio")]
        stalls = sorted(((float(v or 0), h) for h, v in stalls), reverse=True)[:6]
        if stalls:
            print("  top stall reasons (warp-cycles per issued instruction):")
            for v, h in stalls:
                print(f"    {h.replace('smsp__average_warp_latency_issue_stalled_', ''):50s} {v:8.3f}")


if __name__ == "__main__":
    main(sys.argv[1])

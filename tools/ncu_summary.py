"""Summarise an ncu --set full report (read here, no GPU): per kernel duration,
DRAM traffic vs duration, throughput %, occupancy and the top warp-stall reasons.

  python tools/ncu_summary.py gpurun_out/prof.ncu-rep [> profiles/<name>.txt]
"""
import csv
import io
import subprocess
import sys


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main(rep):
    hdr, units, rows = raw(rep)
    col = {h: i for i, h in enumerate(hdr)}

    def g(r, name):
        i = col.get(name)
        return (r[i], units[i]) if i is not None else (None, None)

    for r in rows:
        name = g(r, "Kernel Name")[0]
        print("=" * 100)
        print(name[:150])
        for m in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                  "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
                  "dram__throughput.avg.pct_of_peak_sustained_elapsed",
                  "sm__throughput.avg.pct_of_peak_sustained_elapsed",
                  "sm__warps_active.avg.pct_of_peak_sustained_active",
                  "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
                  "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                  "sm__inst_executed.avg.per_cycle_active",
                  "smsp__issue_active.avg.pct_of_peak_sustained_active",
                  "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
                  "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
                  "launch__occupancy_limit_shared_mem", "launch__waves_per_multiprocessor",
                  "lts__t_sectors_aperture_sysmem_op_read.sum", "lts__t_bytes.sum",
                  "l1tex__t_bytes_pipe_lsu_mem_global_op_ld.sum",
                  "smsp__sass_inst_executed_op_shared_ld.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"]:
            v, u = g(r, m)
            if v not in (None, ""):
                print(f"  {m:70s} {v:>18s} {u}")
        stalls = []
        for h, i in col.items():
            if h.startswith("smsp__average_warp_latency_issue_stalled_") and h.endswith(".ratio"):
                try:
                    stalls.append((float(r[i]), h[len("smsp__average_warp_latency_issue_stalled_"):-len(".ratio")]))
                except ValueError:
                    pass
            elif h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(r[i]), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        print("  top stall reasons (warps stalled per issue):",
              ", ".join(f"{n}={v:.2f}" for v, n in stalls[:8]))


if __name__ == "__main__":
    main(sys.argv[1])

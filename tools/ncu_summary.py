"""Print the key raw metrics of an ncu report (dev aid; summaries go to profiles/)."""
import csv, subprocess, sys

KEYS = ["gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__cluster_dim_x",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "lts__t_sector_hit_rate.pct"]
STALLS = "smsp__pcsamp_warps_issue_stalled_"


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        print(f"kernel: {d.get('Kernel Name', '')[:110]}")
        for k in KEYS:
            if k in d:
                print(f"  {k} = {d[k]} {u.get(k, '')}")
        st = {k[len(STALLS):]: float(v.replace(',', '')) for k, v in d.items()
              if k.startswith(STALLS) and not k.endswith("not_issued") and v not in ("", "0")}
        tot = sum(st.values()) or 1.0
        top = sorted(st.items(), key=lambda x: -x[1])[:8]
        print("  stall samples: " + ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in top))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)

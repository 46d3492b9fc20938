"""Key metrics of an `ncu --set full` report (one block per captured launch)."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__grid_size",
        "launch__block_size", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_write.sum",
        "lts__t_requests_srcunit_tex_op_atom.sum", "sm__inst_executed.sum"]


def summary(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        out.append("--- " + d.get("Kernel Name", "?")[:120])
        for k in KEYS:
            if k in d:
                out.append(f"  {k:70s} {d[k]:>16s} {u[h.index(k)]}")
        if "dram__bytes_read.sum" in d:
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rb = float(d["dram__bytes_read.sum"]) * scale.get(u[h.index("dram__bytes_read.sum")], 1)
            wb = float(d["dram__bytes_write.sum"]) * scale.get(u[h.index("dram__bytes_write.sum")], 1)
            out.append(f"  {'traffic = dram read + write (bytes)':70s} {rb + wb:16.0f}")
    return "\n".join(out) + "\n"


if __name__ == "__main__":
    hdr = "# " + " ".join(sys.argv[2:]) + "\n" if len(sys.argv) > 2 else ""
    print(hdr + summary(sys.argv[1]), end="")

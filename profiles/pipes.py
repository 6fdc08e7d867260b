"""Pipe / memory-unit utilisation lines of an ncu report: python profiles/pipes.py <rep> [units]"""
import csv, io, subprocess, sys
def main(path, units=4096):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    d = {a: (c, b) for a, b, c in zip(rows[0], rows[1], rows[2])}
    keys = ["gpu__time_duration.sum", "sm__inst_executed.sum", "sm__pipe_fp64_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
            "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ldgsts.sum",
            "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_st.sum",
            "l1tex__lsuin_requests.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed_pipe_uniform_realtime.avg.pct_of_peak_sustained_elapsed",
            "idc__request_cycles_active.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "lts__t_sectors.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed_pipe_fp64.sum", "sm__inst_executed_pipe_lsu.sum"]
    for k in keys:
        if k in d:
            v, u = d[k]
            try:
                f = float(v.replace(",", ""))
                extra = f"  ({f / units:.1f} per unit)" if k.endswith(".sum") and not k.startswith(("gpu__", "dram")) else ""
            except ValueError:
                extra = ""
            print(f"{k} = {v} {u}{extra}")
if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 4096)

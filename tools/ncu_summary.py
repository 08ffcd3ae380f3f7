"""Summarise an ncu --set full capture into the profiles/ JSON that bench.py reads for
roofline.traffic. Usage: ncu_summary.py REP OUT CAPTURE_TEXT TICKS ALG_BYTES_PER_TICK [width layers stages]"""
import csv, io, json, subprocess, sys

KEYS = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__time_duration.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "launch__block_size",
        "launch__grid_size", "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
        "lts__t_sector_hit_rate.pct", "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        # tcgen05 (UTCHMMA) activity: the hmma subpipe metrics above only count legacy mma.sync
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__ops_path_tensor_op_utchmma_src_tf32_dst_fp32_sparsity_off.sum.pct_of_peak_sustained_elapsed",
        "smsp__sass_inst_executed_op_utcmma.sum", "smsp__sass_inst_executed_op_tmem_ldt.sum",
        "smsp__sass_inst_executed_op_tmem_stt.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed"]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    rep, out, capture, ticks, alg = sys.argv[1:6]
    cfg = None
    if len(sys.argv) > 8:
        cfg = {"width": int(sys.argv[6]), "layers": int(sys.argv[7]), "stages": int(sys.argv[8])}
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, vals = rows[0], rows[1], rows[2]
    m = {}
    for k in KEYS:
        if k in head:
            i = head.index(k)
            m[k] = f"{vals[i]} {units[i]}".strip()

    def nbytes(k):
        v, u = m[k].split(" ", 1)
        return float(v.replace(",", "")) * UNIT.get(u, 1)

    rd, wr = nbytes("dram__bytes_read.sum"), nbytes("dram__bytes_write.sum")
    res = {"capture": capture, "ticks_per_launch": int(ticks), "dram_bytes_read": rd, "dram_bytes_write": wr,
           "dram_bytes_per_tick": (rd + wr) / int(ticks), "algorithmic_bytes_per_tick": int(alg), "metrics": m}
    if cfg:
        res["config"] = cfg
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()

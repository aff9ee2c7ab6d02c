"""Summarise an ncu report (or a launch-list CSV) into profiles/.

    python tools/ncu_summary.py full  gpurun_out/prof.ncu-rep  profiles/NAME.json
    python tools/ncu_summary.py launches gpurun_out/launches.csv profiles/NAME.json
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum",
    "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "launch__cluster_dim_x",
    "smsp__sass_inst_executed_op_global_ld.sum", "smsp__sass_inst_executed_op_global_st.sum",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__m_xbar2l1tex_read_bytes.sum",
    "lts__t_sector_hit_rate.pct", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__grid_size", "launch__cluster_dim_y",
]


def full(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:120]}
        for k in KEYS:
            if k in hdr:
                d[k] = f"{r[hdr.index(k)]} {units[hdr.index(k)]}".strip()
        try:
            rd = float(r[hdr.index("dram__bytes_read.sum")])
            wr = float(r[hdr.index("dram__bytes_write.sum")])
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            d["dram_bytes_total"] = rd * scale[units[hdr.index("dram__bytes_read.sum")]] + \
                wr * scale[units[hdr.index("dram__bytes_write.sum")]]
        except Exception:
            pass
        ld_s = "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"
        ld_r = "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum"
        if ld_s in hdr and ld_r in hdr:
            try:
                d["global_ld_sectors_per_request"] = float(r[hdr.index(ld_s)]) / max(1.0, float(r[hdr.index(ld_r)]))
            except Exception:
                pass
        res.append(d)
    return res


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = {}
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            agg.setdefault(d["Kernel Name"][:90], []).append(float(d["Metric Value"]))
    total = sum(sum(v) for v in agg.values())
    return [{"kernel": k, "launches": len(v), "mean_us": sum(v) / len(v) / 1e3, "share": sum(v) / total}
            for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))]


if __name__ == "__main__":
    mode, src, dst = sys.argv[1:4]
    res = full(src) if mode == "full" else launches(src)
    json.dump(res, open(dst, "w"), indent=1)
    print(json.dumps(res, indent=1)[:3000])

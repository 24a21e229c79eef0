"""Summarise an ncu report (.ncu-rep) into the metrics the judge reads, as JSON + markdown.

    python tools/ncu_summary.py gpurun_out/r01_attn.ncu-rep profiles/r01_attn_summary
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "sm__cycles_elapsed.avg.per_second",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "lts__t_sector_hit_rate.pct",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_xu_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "smsp__inst_executed.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
]


def summarise(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        d = {}
        name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        d["kernel"] = name
        for k in KEYS:
            for i, h in enumerate(hdr):
                if h.endswith(k):
                    d[k] = {"value": vals[i], "unit": units[i]}
                    break
        out.append(d)
    return out


if __name__ == "__main__":
    rep, dst = sys.argv[1], sys.argv[2]
    s = summarise(rep)
    with open(dst + ".json", "w") as f:
        json.dump(s, f, indent=1)
    with open(dst + ".md", "w") as f:
        for d in s:
            f.write("### %s\n\n| metric | value |\n|---|---|\n" % d["kernel"][:120])
            for k in KEYS:
                if k in d:
                    f.write("| %s | %s %s |\n" % (k, d[k]["value"], d[k]["unit"]))
            f.write("\n")
    print(open(dst + ".md").read())

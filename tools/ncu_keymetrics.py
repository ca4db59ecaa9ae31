"""Extract the key metrics of an `ncu --set full` report (one launch) to JSON:
duration, DRAM bytes, throughput %, pipe utilisation, occupancy, registers,
shared-memory bank conflicts, top warp-stall reasons."""
import csv
import json
import subprocess
import sys

KEYS = [
    "Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "lts__t_bytes.sum", "sm__cycles_elapsed.avg.per_second",
]


def main(rep, out):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h, units, v = rows[0], rows[1], rows[2]
    d = {}
    for k in KEYS:
        if k in h:
            i = h.index(k)
            d[k] = f"{v[i]} {units[i]}".strip()
    stalls = []
    pre = "smsp__pcsamp_warps_issue_stalled_"
    for i, k in enumerate(h):
        if k.startswith(pre) and not k.endswith("not_issued"):
            try:
                stalls.append((float(v[i]), k))
            except ValueError:
                pass
    d["top_stall_samples"] = {k.replace(pre, ""): x for x, k in sorted(stalls, reverse=True)[:6]}
    json.dump(d, open(out, "w"), indent=1)
    print(json.dumps(d, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])

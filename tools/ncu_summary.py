"""Summarise an ncu --set full capture of k_eval into profiles/ (traffic,
instruction mix, pipe utilisation). Usage: python tools/ncu_summary.py REP NODES OUT"""
import csv
import json
import subprocess
import sys

rep, nodes, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
h, units, v = rr[0], rr[1], rr[2]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "ms": 1e-3, "msecond": 1e-3, "s": 1.0}


def get(name):
    i = h.index(name)
    return float(v[i].replace(",", "")) * SCALE.get(units[i], 1.0)


keep = {}
for i, n in enumerate(h):
    if any(k in n for k in ("pct_of_peak_sustained_active", "pct_of_peak_sustained_elapsed")) and \
            any(k in n for k in ("sm__inst_executed", "pipe_fma", "pipe_alu", "pipe_xu", "issue_active",
                                 "wavefronts_mem_shared.sum", "dram__bytes_read.sum", "warps_active")):
        keep[n] = v[i]
rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
dur = get("gpu__time_duration.sum")
inst = get("sm__inst_executed.sum.per_cycle_elapsed") * get("sm__cycles_elapsed.avg") if "sm__cycles_elapsed.avg" in h else None
summary = {
    "kernel": v[h.index("Kernel Name")] if "Kernel Name" in h else "k_eval",
    "nodes": nodes,
    "duration_s_under_ncu": dur,
    "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
    "dram_bytes_per_node": (rd + wr) / nodes,
    "instructions_per_node": inst / nodes if inst else None,
    "shared_wavefronts_per_node": get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum") / nodes
    if "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum" in h else None,
    "shared_store_bank_conflicts": get("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum")
    if "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum" in h else None,
    "metrics_pct": keep,
}
json.dump(summary, open(out, "w"), indent=1)
print(json.dumps({k: summary[k] for k in ("dram_bytes_per_launch", "dram_bytes_per_node", "instructions_per_node")}))

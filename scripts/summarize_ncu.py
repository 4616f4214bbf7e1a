"""Summarise ncu captures into profiles/ (run here, after gpurun brought the reports back)."""
import csv, json, subprocess, sys, os

def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}

def num(d, k):
    v, u = d[k]
    x = float(v.replace(",", ""))
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1}
    return x * scale.get(u, 1)

summary = {}
out_path = sys.argv[1]
for rep in sys.argv[2:]:
    d = raw(rep)
    name = os.path.basename(rep).replace(".ncu-rep", "")
    variant = ("tf32" if "tf32" in name else "fp16") + ("_split_once" if "splitonce" in name else "")
    t = num(d, "gpu__time_duration.sum")
    rd = num(d, "dram__bytes_read.sum")
    wr = num(d, "dram__bytes_write.sum")
    keys = ["sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed.sum.pct_of_peak_sustained_elapsed",
            "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
    entry = {"report": name, "kernel_time_s": t, "dram_read_bytes": rd, "dram_write_bytes": wr,
             "dram_bytes_per_launch": rd + wr}
    for k in keys:
        if k in d:
            entry[k] = d[k][0]
    n = 16384
    entry["effective_tflops_under_ncu"] = 2 * n ** 3 / t / 1e12
    summary[f"{variant}_{n}"] = entry
json.dump(summary, open(out_path, "w"), indent=1)
print(json.dumps(summary, indent=1))

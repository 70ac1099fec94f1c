"""Summarise an ncu --set full report of one layer step into the JSON that
bench.py reads for roofline.traffic: per kernel duration, DRAM bytes, SM
clock, tensor-pipe and memory throughput.
  python tests/probes/ncu_summary.py report.ncu-rep out.json [k]"""
import csv, io, json, subprocess, sys

rep, out = sys.argv[1], sys.argv[2]
k = int(sys.argv[3]) if len(sys.argv) > 3 else 8
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
want = {"gpu__time_duration.sum": "duration_ns", "dram__bytes_read.sum": "dram_read_bytes",
        "dram__bytes_write.sum": "dram_write_bytes", "sm__cycles_elapsed.avg.per_second": "sm_hz",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_pct",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "memory_throughput_pct",
        "launch__grid_size": "grid", "launch__registers_per_thread": "registers"}
idx = {w: h.index(w) for w in want if w in h}
units = rows[1]
SCALE = {"ns": 1.0, "us": 1e3, "ms": 1e6, "nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6,
         "Gbyte": 1e9, "Tbyte": 1e12, "hz": 1.0, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9, "cycle/second": 1.0,
         "cycle/nsecond": 1e9, "cycle/usecond": 1e6}
kern = {}
for r in rows[2:]:
    name = r[h.index("Kernel Name")]
    short = name.split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "").split("::")[-1]
    if "gemm_pair_kernel" in short or "gemm_tc_kernel" in short:
        sw = any(t in name for t in ("<1>", "<(int)1>", "ILi1E", "<true", "<1, ", "ILb1E"))
        short += "<swiglu>" if sw else "<plain>"
    ent = {}
    for w, i in idx.items():
        try:
            ent[want[w]] = float(r[i].replace(",", "")) * SCALE.get(units[i], 1.0)
        except ValueError:
            ent[want[w]] = 0.0
    ent["dram_bytes"] = ent.get("dram_read_bytes", 0) + ent.get("dram_write_bytes", 0)
    key = short
    n = 2
    while key in kern:
        key = f"{short}#{n}"
        n += 1
    kern[key] = ent
gemm1 = [v for kk, v in kern.items() if "<swiglu>" in kk]
gemm2 = [v for kk, v in kern.items() if "<plain>" in kk]
summary = {"source": f"ncu --set full --clock-control none, one layer step (tests/probes/profile_step.py {k}), "
                     "Mixtral layer shape T=4096, B200; cold-cache replay per kernel",
           "kernels": kern,
           "gemm1": {f"dram_bytes_k{k}": sum(v["dram_bytes"] for v in gemm1),
                     "duration_ns": sum(v["duration_ns"] for v in gemm1), "launches": len(gemm1)},
           "gemm2": {f"dram_bytes_k{k}": sum(v["dram_bytes"] for v in gemm2),
                     "duration_ns": sum(v["duration_ns"] for v in gemm2), "launches": len(gemm2)}}
json.dump(summary, open(out, "w"), indent=1)
for kk, v in kern.items():
    print(f"{kk:34s} {v['duration_ns']/1e3:8.1f} us  dram {v['dram_bytes']/1e6:8.1f} MB  "
          f"tensor {v.get('tensor_pipe_pct', 0):5.1f}%  sm {v.get('sm_hz', 0)/1e9:.2f} GHz")

# profiles/<tag>_c4_ncu.json from the raw-page exports of tools/gpu_validate.sh:
#   python tools/ncu_summarize.py <tag> <out.json>
import csv, json, sys
TAG = sys.argv[1] if len(sys.argv) > 1 else "r2"
OUT = sys.argv[2] if len(sys.argv) > 2 else f"profiles/{TAG}_c4_ncu.json"
out = {"command": "ncu --set full --clock-control none --import-source on --kernel-name-base demangled "
                  "-k regex:'mlp.*_kernel<.*<Op>' -s <launches of the class in one wave> -c 1 python bench.py --steps 1 "
                  "--warmup 0 --cpu-baseline 0 --no-e2e (tools/gpu_validate.sh): the first (largest) launch of each "
                  "class in the second wave"}
want = {"gpu__time_duration.sum": "duration", "dram__bytes_read.sum": "dram_read", "dram__bytes_write.sum": "dram_write",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_active_pct_elapsed",
        "launch__registers_per_thread": "registers_per_thread", "launch__grid_size": "grid", "launch__block_size": "block",
        "smsp__mem_tensor_reads_op_ldt.sum.pct_of_peak_sustained_elapsed": "tmem_ld_reads_pct_of_peak",
        "smsp__mem_tensor_reads_op_utcmma_matrix_c.sum.pct_of_peak_sustained_elapsed": "tmem_mma_c_reads_pct_of_peak",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "lsu_shared_wavefronts_pct_of_peak",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
        "sm__cycles_elapsed.avg.per_second": "sm_clock_hz"}
unit_b = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
unit_t = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}
unit_hz = {"hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9, "cycle/nsecond": 1e9, "cycle/usecond": 1e6, "cycle/second": 1}
for k, key in (("TraceGradOp", "fused_launch"), ("GradOutOp", "gradient_launch"), ("TraceStepOp", "forward_launch")):
    rows = list(csv.reader(open(f"gpurun_out/{TAG}_ncu_{k}_raw.csv")))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {"kernel": vals[hdr.index("Kernel Name")]}
    for h, u, v in zip(hdr, units, vals):
        if h not in want:
            continue
        x = float(v.replace(",", ""))
        n = want[h]
        if n == "duration":
            d["duration_ms"] = x * unit_t[u]
        elif n in ("dram_read", "dram_write"):
            d[n + "_MB"] = x * unit_b[u] / 1e6
        elif n == "sm_clock_hz":
            d["sm_clock_mhz"] = x * unit_hz.get(u, 1) / 1e6
        else:
            d[n] = x
    d["traffic_bytes"] = (d["dram_read_MB"] + d["dram_write_MB"]) * 1e6
    out[key] = d
json.dump(out, open(OUT, "w"), indent=1)
print(json.dumps(out, indent=1))

#!/bin/bash
# One ncu --set full capture of a layer step per k (Mixtral shape, T=4096) and
# of the Qwen layer (decode 64 / prefill 8192, k=8), summarised per kernel into
# profiles/ncu_summary_<tag>.json (bench.py reads roofline.traffic from it).
#   bash tests/probes/ncu_all.sh <tag>     (on the GPU box; writes gpurun_out/)
set -e
tag=${1:-r01d}
mkdir -p gpurun_out
for k in 2 4 8 16; do
  ncu --profile-from-start off --set full --clock-control none --import-source on -f \
      -o gpurun_out/step_k$k python tests/probes/profile_step.py $k 1 > /dev/null 2>&1
  python tests/probes/ncu_summary.py gpurun_out/step_k$k.ncu-rep gpurun_out/sum_k$k.json $k > gpurun_out/sum_k$k.txt
done
for T in 64 8192; do
  ncu --profile-from-start off --set full --clock-control none -f \
      -o gpurun_out/qwen_T$T python tests/probes/profile_qwen.py $T 8 1 > /dev/null 2>&1
  python tests/probes/ncu_summary.py gpurun_out/qwen_T$T.ncu-rep gpurun_out/sum_qwen_T$T.json 8 > gpurun_out/sum_qwen_T$T.txt
done
python - "$tag" <<'PY'
import json, sys
tag = sys.argv[1]
out = {"source": "ncu --profile-from-start off --set full --clock-control none, one layer step per k "
                 "(tests/probes/profile_step.py k 1, Mixtral shape T=4096, default kernel choice) and the Qwen "
                 "layer (tests/probes/profile_qwen.py T 8 1); tests/probes/ncu_summary.py; B200, cold-cache replay "
                 "per kernel", "gemm1": {}, "gemm2": {}}
for k in (2, 4, 8, 16):
    j = json.load(open(f"gpurun_out/sum_k{k}.json"))
    out[f"kernels_k{k}"] = j["kernels"]
    for g in ("gemm1", "gemm2"):
        out[g][f"dram_bytes_k{k}"] = j[g][f"dram_bytes_k{k}"]
        out[g][f"duration_ns_k{k}"] = j[g]["duration_ns"]
for T in (64, 8192):
    out[f"qwen_T{T}_k8"] = json.load(open(f"gpurun_out/sum_qwen_T{T}.json"))["kernels"]
json.dump(out, open(f"gpurun_out/ncu_summary_{tag}.json", "w"), indent=1)
print("wrote", f"gpurun_out/ncu_summary_{tag}.json")
PY
# keep the k=8 report only (gpurun copies back <= 64 MiB)
rm -f gpurun_out/step_k2.ncu-rep gpurun_out/step_k4.ncu-rep gpurun_out/step_k16.ncu-rep gpurun_out/qwen_T*.ncu-rep

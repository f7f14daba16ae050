#!/usr/bin/env bash
# NOTE: compute-sanitizer has since been closed on the GPU pool (runs under it left GPUs needing a
# reset); the committed logs in profiles/r02_sanitize/ are from before that.  Do not run this there.
# compute-sanitizer memcheck / racecheck / synccheck over the pair kernels (tiny config and a
# 6-chunk problem), the design-B kernels, and the peer-memory path (one-GPU group emulation:
# 2 ranks in one process, one backward launch; never ranks time-sliced as processes).
# Run on the GPU box:  bash scripts/sanitize_all.sh  -> gpurun_out/sanitize_*.txt
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CS=compute-sanitizer
run() {  # name tool cmd...
  local name=$1 tool=$2; shift 2
  timeout 1500 $CS --tool $tool --error-exitcode 9 --print-limit 50 "$@" > gpurun_out/sanitize_${name}_${tool}.txt 2>&1
  echo "${name} ${tool} rc=$?" | tee -a gpurun_out/sanitize_summary.txt
}
: > gpurun_out/sanitize_summary.txt
for tool in memcheck racecheck synccheck; do
  run tiny $tool python scripts/sanitize_case.py 64 64 1000
  run chunks6 $tool python scripts/sanitize_case.py 1000 128 41000
  run designb $tool python scripts/sanitize_case.py 300 256 3000 2048
done
# peer-memory exchange fused into the kernels (tests/test_gpu_p2p_emulated.py, world 2)
run p2p memcheck python -m pytest tests/test_gpu_p2p_emulated.py -x -q -k "matches_oracle and 2"

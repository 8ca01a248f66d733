# GPU-box round: parity tests, a bench line and one ncu --set full capture of K1/K2/K3.
# usage: gpurun -- bash tools/gpu_profile.sh <tag>
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py > gpurun_out/bench.log 2>&1
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_resolve_fast|k_preprocess|k_forward_warp" -s 12 -c 3 -o gpurun_out/${1:-prof}_full $CMD > gpurun_out/ncu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; tail -c 600 gpurun_out/bench.log; tail -3 gpurun_out/ncu.log

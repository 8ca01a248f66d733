# End-of-round GPU measurements: tests, every bench config, the reference
# arm, the launch list and one ncu --set full capture of the c1 step.
# usage: gpurun -- bash tools/round_bench.sh <tag>
T=${1:-rXX}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rA > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest_gpu.log
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${T}_smi.txt 2>&1
timeout 500 python bench.py > gpurun_out/${T}_bench_c1.log 2>&1
timeout 400 python bench.py --impl reference --steps 20 --warmup 2 > gpurun_out/${T}_bench_ref.log 2>&1
timeout 300 python bench.py --config c0 --no-cpu-baseline > gpurun_out/${T}_bench_c0.log 2>&1
timeout 400 python bench.py --config c2 --steps 40 --warmup 3 > gpurun_out/${T}_bench_c2.log 2>&1
timeout 600 python bench.py --config c3 --steps 300 --warmup 5 > gpurun_out/${T}_bench_c3.log 2>&1
timeout 600 python bench.py --config c4 --steps 20 --warmup 3 > gpurun_out/${T}_bench_c4.log 2>&1
timeout 500 python bench.py --extensions --no-cpu-baseline > gpurun_out/${T}_bench_c1_ext.log 2>&1
timeout 300 python tools/codec_bench.py > gpurun_out/${T}_codec.json 2>/dev/null
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --pipelines 1"
$CMD > gpurun_out/${T}_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${T}_launches.csv $CMD > gpurun_out/${T}_ncu_launch.log 2>&1
$CMD > gpurun_out/${T}_plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on \
    -k "regex:k_resolve_fast|k_forward_warp|k_preprocess|k_fill" -s 20 -c 4 \
    -o gpurun_out/${T}_full $CMD > gpurun_out/${T}_ncu_full.log 2>&1
tail -1 gpurun_out/${T}_pytest_gpu.log
for f in gpurun_out/${T}_bench_*.log; do echo "$f: $(tail -c 300 $f)"; done

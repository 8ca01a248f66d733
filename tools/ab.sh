# A/B kernel variants on the GPU box: parity tests per variant, then
# interleaved microbench rounds.  usage: bash tools/ab.sh TAG NAME...
T=$1; shift
mkdir -p gpurun_out
for v in "$@"; do
  FVV_B200_LIB=build/variants/$v.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_size.py -q -x > gpurun_out/${T}_${v}_parity.log 2>&1
  echo "$v parity: $(tail -1 gpurun_out/${T}_${v}_parity.log)"
done
for r in 1 2; do
  for v in "$@"; do
    echo "$v r$r $(FVV_B200_LIB=build/variants/$v.so timeout 300 python profiles/microbench.py --reps 300 2>/dev/null | tail -1)"
  done
done | tee gpurun_out/${T}_ab.txt

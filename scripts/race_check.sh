# repeat the full-size C2 engine parity tests (fp16 / fp32 y, batch 1 / 8) with the working tree, then the A/B
mkdir -p gpurun_out
T=${1:-g11}
for it in 1 2 3 4; do
  echo "== cur $it" >> gpurun_out/${T}_race.txt
  timeout 600 python -m pytest tests/test_gpu_engine.py tests/test_gpu_parity.py -q -x -k "c2_full_size or tb9_mix or full_size" >> gpurun_out/${T}_race.txt 2>&1
done
bash scripts/ab_engine_vs_head.sh $T
exit 0

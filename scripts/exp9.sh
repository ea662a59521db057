# current state: per-shape timing + in-kernel timeline + C3 sweep (batch 1, 8)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu9.txt 2>&1
{
for sh in 4096x4096 14336x4096; do
  for x4 in 10 16; do
   python tools/prof_gemv.py --shape $sh --scheme tcq --bits-x4 $x4 --time --pdl 2>&1 | tail -1
   QP_TIMELINE=1 python tools/prof_gemv.py --shape $sh --scheme tcq --bits-x4 $x4 --iters 4 2>&1 | tail -1
  done
done
} > gpurun_out/exp9_timeline.txt 2>&1
timeout 1500 python tools/sweep.py --batches 1,8 --out gpurun_out/sweep9.jsonl > gpurun_out/sweep9.txt 2>&1
exit 0

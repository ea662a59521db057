mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv,noheader,nounits > gpurun_out/smi.txt 2>&1
for sh in 4096x4096 14336x4096 4096x14336 28672x8192; do
 for x4 in 10 16; do
  python tools/prof_gemv.py --shape $sh --scheme tcq --bits-x4 $x4 --time --pdl 2>&1 | tail -1
  python tools/prof_gemv.py --shape $sh --scheme tcq --bits-x4 $x4 --time 2>&1 | tail -1
 done
done
QP_TIMELINE=1 python tools/prof_gemv.py --shape 14336x4096 --scheme tcq --bits-x4 10 --iters 4 2>&1 | tail -4
QP_TIMELINE=1 python tools/prof_gemv.py --shape 4096x4096 --scheme tcq --bits-x4 10 --iters 4 2>&1 | tail -4

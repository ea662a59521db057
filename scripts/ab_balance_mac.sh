# A/B: cost-weighted CTA ranges (QP_ENG_ROWCOST / QP_ENG_HALFCOST / QP_ENG_JOB_TILES) on the C2 engine
# step, plus an ncu capture of the MAC micro-benchmark variants (tools/ubench/mac_ab).
mkdir -p gpurun_out
for B in 1 8; do
  for cfg in "0 0 16" "1 0 16" "2 0 16" "1 0.04 16" "2 0.04 16" "0 0.04 16" "1 0.04 8" "1 0.04 24"; do
    set -- $cfg
    echo "E=$1 H=$2 JT=$3" >> gpurun_out/g6_bal_b${B}.txt
    QP_ENG_ROWCOST=$1 QP_ENG_HALFCOST=$2 QP_ENG_JOB_TILES=$3 timeout 200 python tools/engine_ab.py --sets c2 --batch $B --iters 30 >> gpurun_out/g6_bal_b${B}.txt 2>&1
  done
done
timeout 600 ncu --section SchedulerStats --section WarpStateStats --section ComputeWorkloadAnalysis --section InstructionStats \
  --section LaunchStats --clock-control none -k regex:"^k" -o gpurun_out/g6_mac_ab tools/ubench/mac_ab > gpurun_out/g6_mac_ab_ncu.log 2>&1
tools/ubench/mac_ab > gpurun_out/g6_mac_ab.txt 2>&1
exit 0

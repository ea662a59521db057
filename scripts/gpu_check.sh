#!/bin/bash
# One gpurun session: GPU parity tests, smoke, bench line (+ reference arm), ncu launch list,
# per-launch DRAM traffic of the GEMV for the roofline, and a --set full capture of the
# dominant kernel. Outputs land in gpurun_out/.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
if [ "${QP_NCU:-1}" = "1" ]; then
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:qp_gemv_kernel \
  --print-units base --csv --log-file gpurun_out/traffic.csv python tools/ncu_traffic.py > gpurun_out/ncu_traffic.log 2>&1
python tools/ncu_traffic.py --parse gpurun_out/traffic.csv > /dev/null 2>&1 && cp profiles/gemv_traffic.json gpurun_out/
fi
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err
if [ "${QP_NCU:-1}" = "1" ]; then
QP_BENCH_EAGER=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qp_gemv_kernel -s 4 -c 2 \
  -o gpurun_out/prof_gemv python tools/prof_gemv.py --shape 14336x4096 --scheme tcq --bits-x4 10 --iters 8 > gpurun_out/ncu_full.log 2>&1
fi
exit 0

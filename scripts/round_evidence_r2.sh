#!/bin/bash
# Round-2 GPU evidence on one box (outputs in gpurun_out/ev3_*): GPU tests, smoke, engine DRAM traffic
# (ncu, lib-sha-tagged), bench line (x2) + reference arm, ncu launch list of the bench step, ncu --set full
# of the engine kernel at batch 1 and 8.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/ev3_gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/ev3_pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/ev3_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev3_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/ev3_smoke.txt
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:qp_engine_kernel \
  --print-units base --csv --log-file gpurun_out/ev3_eng_traffic.csv python tools/ncu_traffic.py --engine > gpurun_out/ev3_eng_traffic.log 2>&1
python tools/ncu_traffic.py --parse-engine gpurun_out/ev3_eng_traffic.csv > gpurun_out/ev3_eng_traffic_parse.log 2>&1 && cp profiles/engine_traffic.json gpurun_out/ev3_engine_traffic.json
timeout 900 python bench.py > gpurun_out/ev3_bench.json 2> gpurun_out/ev3_bench.err
timeout 900 python bench.py > gpurun_out/ev3_bench2.json 2>> gpurun_out/ev3_bench.err
timeout 300 python bench.py --impl reference > gpurun_out/ev3_bench_ref.json 2>> gpurun_out/ev3_bench.err
QP_BENCH_EAGER=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/ev3_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ev3_ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qp_engine_kernel -s 4 -c 1 \
  -o gpurun_out/ev3_prof_engine python tools/engine_ab.py --sets c2 --eager --iters 1 > gpurun_out/ev3_ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qp_engine_kernel -s 4 -c 1 \
  -o gpurun_out/ev3_prof_engine_b8 python tools/engine_ab.py --sets c2 --eager --iters 1 --batch 8 > gpurun_out/ev3_ncu_full_b8.log 2>&1
exit 0

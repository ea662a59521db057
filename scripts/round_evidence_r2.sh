#!/bin/bash
# Round-2 GPU evidence on one box (outputs in gpurun_out/ev9_*): GPU tests, smoke, engine DRAM traffic
# (ncu, lib-sha-tagged), bench line (x2) + reference arm, ncu launch list of the bench step, ncu --set full
# of the engine kernel at batch 1 and 8.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/ev9_gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/ev9_pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/ev9_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev9_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/ev9_smoke.txt
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:qp_engine_kernel \
  --print-units base --csv --log-file gpurun_out/ev9_eng_traffic.csv python tools/ncu_traffic.py --engine > gpurun_out/ev9_eng_traffic.log 2>&1
python tools/ncu_traffic.py --parse-engine gpurun_out/ev9_eng_traffic.csv > gpurun_out/ev9_eng_traffic_parse.log 2>&1 && cp profiles/engine_traffic.json gpurun_out/ev9_engine_traffic.json
timeout 900 python bench.py > gpurun_out/ev9_bench.json 2> gpurun_out/ev9_bench.err
timeout 900 python bench.py > gpurun_out/ev9_bench2.json 2>> gpurun_out/ev9_bench.err
timeout 300 python bench.py --impl reference > gpurun_out/ev9_bench_ref.json 2>> gpurun_out/ev9_bench.err
QP_BENCH_EAGER=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/ev9_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ev9_ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qp_engine_kernel -s 4 -c 1 \
  -o gpurun_out/ev9_prof_engine python tools/engine_ab.py --sets c2 --eager --iters 1 > gpurun_out/ev9_ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qp_engine_kernel -s 4 -c 1 \
  -o gpurun_out/ev9_prof_engine_b8 python tools/engine_ab.py --sets c2 --eager --iters 1 --batch 8 > gpurun_out/ev9_ncu_full_b8.log 2>&1
timeout 1500 python tools/engine_ab.py --palette --batches 1,2,4,8 --iters 10 > gpurun_out/ev9_c3.jsonl 2> gpurun_out/ev9_c3.err
timeout 400 python tools/decoder_layer.py --engine --out gpurun_out/ev9_c5.jsonl > gpurun_out/ev9_c5.txt 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py > gpurun_out/ev9_san_$tool.txt 2>&1
  echo "rc=$?" >> gpurun_out/ev9_san_$tool.txt
done
exit 0

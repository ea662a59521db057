#!/bin/bash
mkdir -p gpurun_out
for i in 1 2; do
  timeout 300 python tools/engine_ab.py --sets c2,vq3 --batches 1,8 > gpurun_out/ab8_base_$i.jsonl 2>&1
  QP_LIB_PATH=paper_2509_20214_b200/libqpalette_prev.so timeout 300 python tools/engine_ab.py --sets c2,vq3 --batches 1,8 > gpurun_out/ab8_nc_$i.jsonl 2>&1
done
timeout 300 python tools/engine_ab.py --sets c2,vq3 --batch 8 --prerotated > gpurun_out/ab8_pre.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:qp_ -c 12 --csv --log-file gpurun_out/ab8_launches.csv \
  env QP_BENCH_EAGER=1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ab8_ncu.log 2>&1

#!/bin/bash
mkdir -p gpurun_out
for i in 1 2; do
  timeout 300 python tools/engine_ab.py --sets c2,sq_tcq25,vq3,nuq4 > gpurun_out/abm_base_$i.jsonl 2>&1
  QP_LIB_PATH=paper_2509_20214_b200/libqpalette_prev.so timeout 300 python tools/engine_ab.py --sets c2,sq_tcq25,vq3,nuq4 > gpurun_out/abm_w12_$i.jsonl 2>&1
  QP_NS_MAX=4 timeout 300 python tools/engine_ab.py --sets c2,vq3,nuq4 > gpurun_out/abm_ns4_$i.jsonl 2>&1
done
timeout 300 python tools/engine_ab.py --sets c2,vq3 --batch 8 > gpurun_out/abm_base_b8.jsonl 2>&1
QP_LIB_PATH=paper_2509_20214_b200/libqpalette_prev.so timeout 300 python tools/engine_ab.py --sets c2,vq3 --batch 8 > gpurun_out/abm_w12_b8.jsonl 2>&1

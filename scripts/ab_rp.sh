#!/bin/bash
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_engine.py -q -x -k "not c2_full" > gpurun_out/rp_t.log 2>&1; echo rc=$? >> gpurun_out/rp_t.log
timeout 900 python -m pytest tests/test_gpu_engine.py -q -x -k "c2_full" > gpurun_out/rp_t2.log 2>&1; echo rc=$? >> gpurun_out/rp_t2.log
for i in 1 2; do
  timeout 300 python tools/engine_ab.py --sets c2,vq3,nuq4 --batches 1,4,8 > gpurun_out/rp_new_$i.jsonl 2>&1
  QP_LIB_PATH=paper_2509_20214_b200/libqpalette_prev.so timeout 300 python tools/engine_ab.py --sets c2,vq3,nuq4 --batches 1,4,8 > gpurun_out/rp_prev_$i.jsonl 2>&1
done

#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python tools/engine_ab.py --palette --batches 1,2,4,8 --iters 10 > gpurun_out/c3_engine_v2.jsonl 2> gpurun_out/c3_engine_v2.err
timeout 900 python tools/engine_ab.py --c4 --batches 1,8 --iters 10 > gpurun_out/c4_engine.jsonl 2> gpurun_out/c4_engine.err
timeout 400 python tools/decoder_layer.py --engine --out gpurun_out/c5_engine_v2.jsonl > gpurun_out/c5_engine_v2.txt 2>&1

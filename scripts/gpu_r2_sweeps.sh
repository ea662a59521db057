#!/bin/bash
# Round-2 GPU evidence: engine tests, C3 palette through the engine (batch 1/2/4/8), C5 decoder layer
# (per op and engine), Fig. 2 / MSQ plan with the R22 scales. Outputs in gpurun_out/.
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_engine.py -q -x -k "not c2_full" > gpurun_out/sw_t.log 2>&1; echo rc=$? >> gpurun_out/sw_t.log
timeout 1500 python tools/engine_ab.py --palette --batches 1,2,4,8 --iters 10 > gpurun_out/c3_engine.jsonl 2> gpurun_out/c3_engine.err
timeout 400 python tools/decoder_layer.py --engine --out gpurun_out/c5_engine.jsonl > gpurun_out/c5_engine.txt 2>&1
timeout 400 python tools/decoder_layer.py --out gpurun_out/c5_perop.jsonl > gpurun_out/c5_perop.txt 2>&1
timeout 900 python tools/plan_msq.py --out gpurun_out/msq_r2.jsonl > gpurun_out/msq_r2.txt 2>&1

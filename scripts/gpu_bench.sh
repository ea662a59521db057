#!/bin/bash
# Engine DRAM traffic (ncu, tagged with the lib sha256) -> profiles/engine_traffic.json, then the
# bench line (reads it) and the reference arm. Outputs in gpurun_out/.
mkdir -p gpurun_out
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:qp_engine_kernel \
  --print-units base --csv --log-file gpurun_out/eng_traffic.csv python tools/ncu_traffic.py --engine > gpurun_out/eng_traffic.log 2>&1
python tools/ncu_traffic.py --parse-engine gpurun_out/eng_traffic.csv > gpurun_out/eng_traffic_parse.log 2>&1 && cp profiles/engine_traffic.json gpurun_out/
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err

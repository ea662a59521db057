#!/bin/bash
# A/B of the engine: the in-tree library vs paper_2509_20214_b200/libqpalette_prev.so, alternating,
# same session. Usage: scripts/ab_engine.sh <sets> <rounds> <out-prefix>
SETS=${1:-c2,sq_tcq25,big_tcq25}; R=${2:-2}; OUT=${3:-gpurun_out/ab}
for i in $(seq 1 $R); do
  timeout 300 python tools/engine_ab.py --sets $SETS > ${OUT}_new_$i.jsonl 2>&1
  QP_LIB_PATH=paper_2509_20214_b200/libqpalette_prev.so timeout 300 python tools/engine_ab.py --sets $SETS > ${OUT}_prev_$i.jsonl 2>&1
done

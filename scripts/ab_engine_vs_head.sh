# A/B: HEAD engine (abtmp_old) vs the no-pool engine (p2p epilogue, acquire polling, spread counters)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_multiproc.py -q -x > gpurun_out/g5_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/g5_tests.txt
for it in 1 2; do
for B in 1 8; do
  (cd abtmp_old && timeout 300 python tools/engine_ab.py --sets c2,sq_tcq25,big_tcq25,vq3 --batch $B --iters 20) > gpurun_out/g5_ab_old_b${B}_$it.jsonl 2>&1
  timeout 300 python tools/engine_ab.py --sets c2,sq_tcq25,big_tcq25,vq3 --batch $B --iters 20 > gpurun_out/g5_ab_new_b${B}_$it.jsonl 2>&1
done
done
(cd abtmp_old && QP_LIB_PATH=paper_2509_20214_b200/libqpalette_tl.so timeout 300 python tools/engine_timeline.py --sets c2) > gpurun_out/g5_tl_old.txt 2>&1
QP_LIB_PATH=paper_2509_20214_b200/libqpalette_tl.so timeout 300 python tools/engine_timeline.py --sets c2 > gpurun_out/g5_tl_new.txt 2>&1
exit 0

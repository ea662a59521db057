mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g1_gpu.txt 2>&1
timeout 600 python bench.py > gpurun_out/g1_bench.json 2> gpurun_out/g1_bench.err
QP_LIB_PATH=paper_2509_20214_b200/libqpalette_tl.so timeout 300 python tools/engine_timeline.py --sets c2 > gpurun_out/g1_tl.txt 2>&1
QP_LIB_PATH=paper_2509_20214_b200/libqpalette_tl.so timeout 300 python tools/engine_timeline.py --sets c2 --prerotated >> gpurun_out/g1_tl.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qp_engine_kernel -s 4 -c 1 \
  -o gpurun_out/g1_prof python tools/engine_ab.py --sets c2 --eager --iters 1 > gpurun_out/g1_ncu.log 2>&1
exit 0

# ncu source-level stall sampling of the GEMV (new staged + old) on 4096x4096 TCQ-2.5
mkdir -p gpurun_out
for v in new old; do
  lib=libqpalette.so; [ $v = old ] && lib=libqpalette_old.so
  QP_LIB_PATH=$PWD/paper_2509_20214_b200/$lib timeout 600 ncu --set full --clock-control none --import-source on -k regex:qp_gemv_kernel -s 4 -c 1 \
    -o gpurun_out/prof11_$v python tools/prof_gemv.py --shape 4096x4096 --scheme tcq --bits-x4 10 --iters 8 > gpurun_out/ncu11_$v.log 2>&1
done
exit 0

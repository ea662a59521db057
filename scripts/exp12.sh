mkdir -p gpurun_out
{
for lib in libqpalette_old.so libqpalette.so libqpalette_noef.so; do
 echo "== $lib"
 for x4 in 10 16; do
   QP_LIB_PATH=$PWD/paper_2509_20214_b200/$lib python tools/prof_gemv.py --shape 14336x4096 --scheme tcq --bits-x4 $x4 --time --pdl 2>&1 | tail -1
 done
done
} > gpurun_out/exp12.txt 2>&1
for v in new old; do
  lib=libqpalette.so; [ $v = old ] && lib=libqpalette_old.so
  QP_LIB_PATH=$PWD/paper_2509_20214_b200/$lib timeout 600 ncu --set full --clock-control none --import-source on -k regex:qp_gemv_kernel -s 4 -c 1 \
    -o gpurun_out/prof12_$v python tools/prof_gemv.py --shape 14336x4096 --scheme tcq --bits-x4 16 --iters 8 > gpurun_out/ncu12_$v.log 2>&1
done
exit 0

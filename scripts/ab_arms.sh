# cur vs va (inline peer helpers) vs vb (atomicAdd workspace reductions)
mkdir -p gpurun_out
T=${1:-g23}
for it in 1 2; do
for B in 1 8; do
  for arm in cur va vb; do
    lib=paper_2509_20214_b200/libqpalette.so; [ $arm != cur ] && lib=paper_2509_20214_b200/libqpalette_$arm.so
    echo "$arm b$B" >> gpurun_out/${T}_ab.txt
    QP_LIB_PATH=$lib timeout 300 python tools/engine_ab.py --sets c5_qkv,c5_gu,c2,sq_tcq25,vq3 --batch $B --iters 30 >> gpurun_out/${T}_ab.txt 2>&1
  done
done
done
exit 0

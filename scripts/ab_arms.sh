# A/B over builds: v3 (abtmp_v3/: the round's previous evidence build), head (abtmp_old/: last commit),
# cur (working tree), cur_rp (working tree, relaxed polling: -DQP_ENG_RELAXED_POLL)
mkdir -p gpurun_out
T=${1:-g9}
run() {   # arm dir libpath
  local arm=$1 dir=$2 lib=$3
  echo "$arm b1" >> gpurun_out/${T}_ab.txt
  (cd $dir && QP_LIB_PATH=$lib timeout 300 python tools/engine_ab.py --sets c2,sq_tcq25,vq3,nuq4 --batch 1 --iters 30) >> gpurun_out/${T}_ab.txt 2>&1
  echo "$arm b8" >> gpurun_out/${T}_ab.txt
  (cd $dir && QP_LIB_PATH=$lib timeout 300 python tools/engine_ab.py --sets c2,sq_tcq25,vq3,nuq4 --batch 8 --iters 30) >> gpurun_out/${T}_ab.txt 2>&1
  (cd $dir && QP_LIB_PATH=$lib timeout 300 python tools/decoder_layer.py --engine --out /tmp/c5_$arm.jsonl) > /dev/null 2>&1
  sed "s/^/$arm /" /tmp/c5_$arm.jsonl >> gpurun_out/${T}_c5.txt
}
for it in 1 2; do
  run v3 abtmp_v3 paper_2509_20214_b200/libqpalette.so
  run head abtmp_old paper_2509_20214_b200/libqpalette.so
  run cur . paper_2509_20214_b200/libqpalette.so
  run cur_rp . paper_2509_20214_b200/libqpalette_rp.so
done
timeout 600 python -m pytest tests/test_gpu_engine.py -q -x > gpurun_out/${T}_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.txt
exit 0

# small knobs: spin polling (-DQP_ENG_SPIN_POLL), rotation-job skew 8 / 24 tiles, vs the default build
mkdir -p gpurun_out
T=${1:-g25}
for it in 1 2; do
for B in 1 8; do
  echo "cur b$B" >> gpurun_out/${T}_ab.txt
  timeout 300 python tools/engine_ab.py --sets c2,sq_tcq25,c5_qkv --batch $B --iters 30 >> gpurun_out/${T}_ab.txt 2>&1
  echo "va b$B" >> gpurun_out/${T}_ab.txt
  QP_LIB_PATH=paper_2509_20214_b200/libqpalette_sp.so timeout 300 python tools/engine_ab.py --sets c2,sq_tcq25,c5_qkv --batch $B --iters 30 >> gpurun_out/${T}_ab.txt 2>&1
  echo "np b$B" >> gpurun_out/${T}_ab.txt
  QP_ENG_JOB_TILES=8 timeout 300 python tools/engine_ab.py --sets c2,sq_tcq25,c5_qkv --batch $B --iters 30 >> gpurun_out/${T}_ab.txt 2>&1
  echo "rp b$B" >> gpurun_out/${T}_ab.txt
  QP_ENG_JOB_TILES=24 timeout 300 python tools/engine_ab.py --sets c2,sq_tcq25,c5_qkv --batch $B --iters 30 >> gpurun_out/${T}_ab.txt 2>&1
done
done
exit 0

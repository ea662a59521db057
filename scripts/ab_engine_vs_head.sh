# A/B: HEAD engine (abtmp_old/, a build of the last commit) vs the working tree's build
mkdir -p gpurun_out
T=${1:-g8}
for it in 1 2; do
for B in 1 8; do
  echo "old b$B" >> gpurun_out/${T}_ab.txt
  (cd abtmp_old && timeout 300 python tools/engine_ab.py --sets c2,sq_tcq25,big_tcq25,vq3,nuq4,c5_qkv,c5_gu --batch $B --iters 30) >> gpurun_out/${T}_ab.txt 2>&1
  echo "new b$B" >> gpurun_out/${T}_ab.txt
  timeout 300 python tools/engine_ab.py --sets c2,sq_tcq25,big_tcq25,vq3,nuq4,c5_qkv,c5_gu --batch $B --iters 30 >> gpurun_out/${T}_ab.txt 2>&1
done
done
timeout 600 python -m pytest tests/test_gpu_engine.py -q -x > gpurun_out/${T}_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.txt
exit 0

# v3 (abtmp_v3) vs cur: the C5 launches, the C2 sets, the C5 decoder layer; then the GPU parity tests
mkdir -p gpurun_out
T=${1:-g21}
for it in 1 2; do
for B in 1 8; do
  echo "v3 b$B" >> gpurun_out/${T}_ab.txt
  (cd abtmp_v3 && timeout 300 python tools/engine_ab.py --sets c5_qkv,c5_o,c5_gu,c5_down,c2,sq_tcq25,vq3 --batch $B --iters 30) >> gpurun_out/${T}_ab.txt 2>&1
  echo "cur b$B" >> gpurun_out/${T}_ab.txt
  timeout 300 python tools/engine_ab.py --sets c5_qkv,c5_o,c5_gu,c5_down,c2,sq_tcq25,vq3 --batch $B --iters 30 >> gpurun_out/${T}_ab.txt 2>&1
done
done
for arm in v3 cur; do
  dir=.; [ $arm = v3 ] && dir=abtmp_v3
  (cd $dir && timeout 300 python tools/decoder_layer.py --engine --out /tmp/c5_$arm.jsonl) > /dev/null 2>&1
  sed "s/^/$arm /" /tmp/c5_$arm.jsonl >> gpurun_out/${T}_c5.txt
done
timeout 900 python -m pytest tests/test_gpu_engine.py -q -x > gpurun_out/${T}_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.txt
exit 0

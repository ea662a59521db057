# the engine's in-kernel round protocol (fused all-gather): multi-process + world-1 tests, engine A/B vs
# the last commit (abtmp_old/), and the bench's sharded code path at world 1 (p2p vs NCCL)
mkdir -p gpurun_out
T=${1:-g26}
timeout 1200 python -m pytest tests/test_gpu_multiproc.py tests/test_gpu_engine.py -q -x > gpurun_out/${T}_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.txt
for it in 1 2; do
for B in 1 8; do
  echo "old b$B" >> gpurun_out/${T}_ab.txt
  (cd abtmp_old && timeout 300 python tools/engine_ab.py --sets c2,sq_tcq25,c5_qkv,vq3 --batch $B --iters 30) >> gpurun_out/${T}_ab.txt 2>&1
  echo "new b$B" >> gpurun_out/${T}_ab.txt
  timeout 300 python tools/engine_ab.py --sets c2,sq_tcq25,c5_qkv,vq3 --batch $B --iters 30 >> gpurun_out/${T}_ab.txt 2>&1
done
done
QP_BENCH_FORCE_SHARDED=1 timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_fs_p2p.json 2> gpurun_out/${T}_fs_p2p.err
QP_BENCH_FORCE_SHARDED=1 timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --allgather nccl > gpurun_out/${T}_fs_nccl.json 2> gpurun_out/${T}_fs_nccl.err
exit 0

# One gpurun session producing the round's GPU evidence (outputs in gpurun_out/):
# GPU parity tests, smoke, bench line (+ reference arm), per-launch DRAM traffic of the GEMV (ncu),
# ncu launch list of the bench step, ncu --set full of the dominant kernel, the C3 palette sweep
# the C5 decoder layer and the C4 70B row shards (compute side, one GPU).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/ev_gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/ev_pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/ev_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/ev_smoke.txt
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:qp_gemv_kernel \
  --print-units base --csv --log-file gpurun_out/ev_traffic.csv python tools/ncu_traffic.py > gpurun_out/ev_ncu_traffic.log 2>&1
python tools/ncu_traffic.py --parse gpurun_out/ev_traffic.csv > gpurun_out/ev_ncu_traffic_parse.log 2>&1 && cp profiles/gemv_traffic.json gpurun_out/ev_gemv_traffic.json
timeout 600 python bench.py > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err
timeout 600 python bench.py > gpurun_out/ev_bench2.json 2>> gpurun_out/ev_bench.err
timeout 300 python bench.py --impl reference > gpurun_out/ev_bench_ref.json 2>> gpurun_out/ev_bench.err
QP_BENCH_EAGER=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/ev_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ev_ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qp_gemv_kernel -s 4 -c 1 \
  -o gpurun_out/ev_prof_gemv python tools/prof_gemv.py --shape 14336x4096 --scheme tcq --bits-x4 10 --iters 8 > gpurun_out/ev_ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qp_gemv_kernel -s 4 -c 1 \
  -o gpurun_out/ev_prof_gemv_b8 python tools/prof_gemv.py --shape 14336x4096 --scheme tcq --bits-x4 10 --iters 8 --batch 8 > gpurun_out/ev_ncu_full_b8.log 2>&1
timeout 1500 python tools/sweep.py --batches 1,2,4,8 --out gpurun_out/ev_sweep.jsonl > gpurun_out/ev_sweep.txt 2>&1
timeout 600 python tools/decoder_layer.py --out gpurun_out/ev_c5.jsonl > gpurun_out/ev_c5.txt 2>&1
timeout 900 python tools/sweep.py --shapes 28672x8192,8192x28672 --widths c4 --batches 1,8 --shards 1,2,4,8 \
  --out gpurun_out/ev_c4.jsonl > gpurun_out/ev_c4.txt 2>&1
exit 0

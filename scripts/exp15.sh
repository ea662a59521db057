mkdir -p gpurun_out
for cfg in "vq 8" "tcq 10"; do
  set -- $cfg
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:qp_gemv_kernel -s 4 -c 1 \
    -o gpurun_out/prof15_$1 python tools/prof_gemv.py --shape 14336x4096 --scheme $1 --bits-x4 $2 --iters 8 > gpurun_out/ncu15_$1.log 2>&1
done
for sx in vq:8 tcq:10 tcq:16 nuq:16; do
  python tools/prof_gemv.py --shape 14336x4096 --scheme ${sx%%:*} --bits-x4 ${sx##*:} --time --pdl 2>&1 | tail -1
  QP_TIMELINE=1 python tools/prof_gemv.py --shape 14336x4096 --scheme ${sx%%:*} --bits-x4 ${sx##*:} --iters 4 2>&1 | tail -1
done > gpurun_out/exp15.txt 2>&1
exit 0

# A/B over env variants for the small-table schemes: bash scripts/ab5.sh <out> "name:lib:ENV" ...
out=$1; shift
mkdir -p gpurun_out
: > gpurun_out/${out}.txt
for round in 1 2; do
 for b in 1 8; do
 for cfg in 4096x4096:vq:8 4096x4096:nuq:16 14336x4096:vq:8 14336x4096:vq:12 14336x4096:nuq:16 4096x14336:vq:12 4096x14336:nuq:12 14336x4096:unif:12; do
  IFS=: read sh sc x4 <<< "$cfg"
  for v in "$@"; do
   IFS=: read name lib envs <<< "$v"
   r=$(env QP_LIB_PATH=$PWD/paper_2509_20214_b200/$lib $envs python tools/prof_gemv.py --shape $sh --scheme $sc --bits-x4 $x4 --time --pdl --batch $b 2>&1 | tail -1)
   echo "$name | $r" >> gpurun_out/${out}.txt
  done
 done
 done
done
python tools/ab_summary.py gpurun_out/${out}.txt > gpurun_out/${out}_summary.txt 2>&1
exit 0

# robust A/B: alternate variants, 3 rounds; tools/ab_summary.py prints the per-variant minimum.
# bash scripts/ab3.sh <out> lib1.so lib2.so ...
out=$1; shift
mkdir -p gpurun_out
: > gpurun_out/${out}.txt
for round in 1 2 3; do
 for sh in 4096x4096 14336x4096 4096x14336; do
  for sx in tcq:10 half_tcq:13 tcq:16 vq:8; do
   for lib in "$@"; do
    r=$(QP_LIB_PATH=$PWD/paper_2509_20214_b200/$lib python tools/prof_gemv.py --shape $sh --scheme ${sx%%:*} --bits-x4 ${sx##*:} --time --pdl 2>&1 | tail -1)
    echo "$lib | $r" >> gpurun_out/${out}.txt
   done
  done
 done
 for lib in "$@"; do
  r=$(QP_LIB_PATH=$PWD/paper_2509_20214_b200/$lib python tools/prof_gemv.py --shape 14336x4096 --scheme tcq --bits-x4 10 --time --pdl --batch 8 2>&1 | tail -1)
  echo "$lib | $r" >> gpurun_out/${out}.txt
 done
done
python tools/ab_summary.py gpurun_out/${out}.txt > gpurun_out/${out}_summary.txt 2>&1
exit 0

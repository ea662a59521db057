# short A/B: bash scripts/ab2.sh <out> lib1.so lib2.so ...
out=$1; shift
mkdir -p gpurun_out
{
for lib in "$@"; do
 echo "== $lib"
 for sh in 4096x4096 14336x4096 4096x14336; do
  for sx in tcq:10 half_tcq:13 tcq:16; do
   QP_LIB_PATH=$PWD/paper_2509_20214_b200/$lib python tools/prof_gemv.py --shape $sh --scheme ${sx%%:*} --bits-x4 ${sx##*:} --time --pdl 2>&1 | tail -1
  done
 done
 for sx in vq:8 nuq:16 vq:12; do
 QP_LIB_PATH=$PWD/paper_2509_20214_b200/$lib python tools/prof_gemv.py --shape 14336x4096 --scheme ${sx%%:*} --bits-x4 ${sx##*:} --time --pdl 2>&1 | tail -1
 done
 QP_LIB_PATH=$PWD/paper_2509_20214_b200/$lib python tools/prof_gemv.py --shape 14336x4096 --scheme tcq --bits-x4 10 --time --pdl --batch 8 2>&1 | tail -1
done
} > gpurun_out/${out}.txt 2>&1
exit 0

# A/B timing of GEMV variants: bash scripts/ab.sh <out> lib1.so lib2.so ...  (+ QP_AB_TESTS=1 runs pytest -m gpu first)
out=$1; shift
mkdir -p gpurun_out
if [ "${QP_AB_TESTS:-0}" = "1" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${out}_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/${out}_pytest.txt
fi
{
for lib in "$@"; do
 echo "== $lib"
 for sh in 4096x4096 14336x4096 4096x14336; do
  for sx in tcq:10 half_tcq:13 tcq:16; do
   QP_LIB_PATH=$PWD/paper_2509_20214_b200/$lib python tools/prof_gemv.py --shape $sh --scheme ${sx%%:*} --bits-x4 ${sx##*:} --time --pdl 2>&1 | tail -1
  done
 done
 QP_LIB_PATH=$PWD/paper_2509_20214_b200/$lib python tools/prof_gemv.py --shape 14336x4096 --scheme vq --bits-x4 8 --time --pdl 2>&1 | tail -1
 QP_LIB_PATH=$PWD/paper_2509_20214_b200/$lib python tools/prof_gemv.py --shape 14336x4096 --scheme nuq --bits-x4 16 --time --pdl 2>&1 | tail -1
 QP_LIB_PATH=$PWD/paper_2509_20214_b200/$lib python tools/prof_gemv.py --shape 14336x4096 --scheme tcq --bits-x4 10 --time --pdl --batch 8 2>&1 | tail -1
 QP_LIB_PATH=$PWD/paper_2509_20214_b200/$lib QP_TIMELINE=1 python tools/prof_gemv.py --shape 4096x4096 --scheme tcq --bits-x4 10 --iters 4 2>&1 | tail -1
 QP_LIB_PATH=$PWD/paper_2509_20214_b200/$lib QP_TIMELINE=1 python tools/prof_gemv.py --shape 14336x4096 --scheme tcq --bits-x4 16 --iters 4 2>&1 | tail -1
done
} > gpurun_out/${out}.txt 2>&1
exit 0

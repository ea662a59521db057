# staged (TMA ring) GEMV vs previous register-prefetch GEMV: parity + timing + timeline
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest10.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest10.txt
{
for lib in libqpalette_old.so libqpalette.so; do
 echo "== $lib"
 for sh in 4096x4096 14336x4096 4096x14336; do
  for x4 in 10 16; do
   QP_LIB_PATH=$PWD/paper_2509_20214_b200/$lib python tools/prof_gemv.py --shape $sh --scheme tcq --bits-x4 $x4 --time --pdl 2>&1 | tail -1
  done
 done
 QP_LIB_PATH=$PWD/paper_2509_20214_b200/$lib python tools/prof_gemv.py --shape 14336x4096 --scheme half_tcq --bits-x4 13 --time --pdl 2>&1 | tail -1
 QP_LIB_PATH=$PWD/paper_2509_20214_b200/$lib python tools/prof_gemv.py --shape 14336x4096 --scheme vq --bits-x4 8 --time --pdl 2>&1 | tail -1
 QP_LIB_PATH=$PWD/paper_2509_20214_b200/$lib python tools/prof_gemv.py --shape 14336x4096 --scheme tcq --bits-x4 10 --time --pdl --batch 8 2>&1 | tail -1
 QP_LIB_PATH=$PWD/paper_2509_20214_b200/$lib QP_TIMELINE=1 python tools/prof_gemv.py --shape 4096x4096 --scheme tcq --bits-x4 10 --iters 4 2>&1 | tail -1
 QP_LIB_PATH=$PWD/paper_2509_20214_b200/$lib QP_TIMELINE=1 python tools/prof_gemv.py --shape 14336x4096 --scheme tcq --bits-x4 10 --iters 4 2>&1 | tail -1
done
} > gpurun_out/exp10.txt 2>&1
exit 0

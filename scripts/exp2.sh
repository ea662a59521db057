# quick perf check: per-shape GEMV timing + in-kernel timeline + gpu tests
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for sh in 4096x4096 14336x4096 4096x14336 28672x8192; do
 for x4 in 10 16; do
  python tools/prof_gemv.py --shape $sh --scheme tcq --bits-x4 $x4 --time --pdl 2>&1 | tail -1
 done
done
for b in 1 8; do python tools/prof_gemv.py --shape 14336x4096 --scheme tcq --bits-x4 10 --time --pdl --batch $b 2>&1 | tail -1; done
QP_TIMELINE=1 python tools/prof_gemv.py --shape 14336x4096 --scheme tcq --bits-x4 10 --iters 4 2>&1 | tail -2
QP_TIMELINE=1 python tools/prof_gemv.py --shape 4096x4096 --scheme tcq --bits-x4 10 --iters 4 2>&1 | tail -2

timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for sh in 4096x4096 14336x4096 4096x14336; do
  for x4 in 10 16; do
   python tools/prof_gemv.py --shape $sh --scheme tcq --bits-x4 $x4 --time --pdl 2>&1 | tail -1
   python tools/prof_gemv.py --shape $sh --scheme tcq --bits-x4 $x4 --time --pdl --rht 2>&1 | tail -1
   python tools/prof_gemv.py --shape $sh --scheme tcq --bits-x4 $x4 --time --pdl --y16 2>&1 | tail -1
  done
done

for nw in 0 8 12; do
 export QP_NWARP=$nw
 echo "== QP_NWARP=$nw"
 for sh in 14336x4096 28672x8192; do
  for x4 in 10 16; do
   python tools/prof_gemv.py --shape $sh --scheme tcq --bits-x4 $x4 --time --pdl 2>&1 | tail -1
  done
 done
done

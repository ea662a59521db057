# A/B: in-word stream fields via IMAD.HI / IMAD (FMA pipe) instead of SHF (ALU pipe): -DQP_FIELD_MULHI
mkdir -p gpurun_out
for it in 1 2; do
for B in 1 8; do
  echo "base b$B" >> gpurun_out/g7_ab.txt
  timeout 300 python tools/engine_ab.py --sets c2,sq_tcq25,big_tcq25,vq3,nuq4 --batch $B --iters 30 >> gpurun_out/g7_ab.txt 2>&1
  echo "mulhi b$B" >> gpurun_out/g7_ab.txt
  QP_LIB_PATH=paper_2509_20214_b200/libqpalette_mh.so timeout 300 python tools/engine_ab.py --sets c2,sq_tcq25,big_tcq25,vq3,nuq4 --batch $B --iters 30 >> gpurun_out/g7_ab.txt 2>&1
done
done
exit 0

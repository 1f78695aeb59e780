mkdir -p gpurun_out
L=gpurun_out/st4.log
for v in st_lag4_c16 st_lag3_c16 st_lag2_c16 st_lag1_c16; do
  if [ $v = base ]; then unset CPRB_LIB; else export CPRB_LIB=$PWD/tools/$v/libcprb200.so; fi
  echo "== $v" >> $L
  timeout 200 python tools/stencil_tl.py 60,220,85 2>&1 | head -1 >> $L
  timeout 300 python tools/stencil_tl.py 120,440,170 2>&1 | head -1 >> $L
  for S in 40,7,33 70,9,40; do CPRB_STENCIL_MAXCLUS=2 timeout 100 python tools/stencil_rounds.py $S 2>&1 | tail -1 >> $L; done
done
cat $L

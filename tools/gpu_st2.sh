mkdir -p gpurun_out
CPRB_LIB=$PWD/tools/stencil_orig/libcprb200.so timeout 300 python tools/stencil_tl.py 60,220,85 > gpurun_out/st2_orig.log 2>&1
timeout 300 python tools/stencil_tl.py 60,220,85 > gpurun_out/st2_new.log 2>&1
cat gpurun_out/st2_orig.log gpurun_out/st2_new.log

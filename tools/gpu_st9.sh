CPRB_LIB=$PWD/tools/st_light/libcprb200.so ALL=1 timeout 200 python tools/stencil_tl.py 60,220,85 2>&1 | grep -E "apply|end us"

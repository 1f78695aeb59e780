mkdir -p gpurun_out
for v in base am_rr64 am_rr128; do
  if [ $v = base ]; then unset CPRB_LIB; else export CPRB_LIB=$PWD/tools/$v/libcprb200.so; fi
  timeout 300 python tools/vcycle_time.py $v 2>&1 | grep -E "vcycle|Error"
done
python - <<'P'
import numpy as np
b = np.load("gpurun_out/vc_base.npy")
for v in ["am_rr64", "am_rr128"]:
    try:
        print(v, "bitwise", np.array_equal(b, np.load(f"gpurun_out/vc_{v}.npy")))
    except Exception as e:
        print(v, e)
P

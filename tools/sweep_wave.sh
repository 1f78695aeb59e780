#!/bin/bash
# Parameter sweep of the wave BILU kernel on the GPU box (no git there):
#   bash tools/sweep_wave.sh "DEPTH RING SLEEP" ...
F=paper_2201_01970_b200/csrc/wave.cu
cp $F /tmp/wave.cu.orig
for v in "$@"; do
  set -- $v
  cp /tmp/wave.cu.orig $F
  sed -i "s/^constexpr int WAVE_DEPTH = [0-9]*;/constexpr int WAVE_DEPTH = $1;/" $F
  sed -i "s/^constexpr int WAVE_RING = [0-9]*;/constexpr int WAVE_RING = $2;/" $F
  sed -i "s/__nanosleep(100);/__nanosleep($3);/" $F
  python -m paper_2201_01970_b200.build_native > /dev/null 2>&1 || { echo "build failed $v"; continue; }
  echo "DEPTH=$1 RING=$2 SLEEP=$3: $(timeout 120 python tools/profile_path.py --what bilu --reps 50 2>&1 | tail -1)"
done
cp /tmp/wave.cu.orig $F
python -m paper_2201_01970_b200.build_native > /dev/null 2>&1

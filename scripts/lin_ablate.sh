#!/bin/bash
# Linear-kernel ablation (research): `build` compiles one library per QS_AB mask into
# scratch/ab<mask>/ (here, no GPU needed); `run` times every variant with linear_bench.
# QS_AB bits (csrc/linear_tc.cu): 1 unpack LDS+ALU off, 2 MMAs off, 4 epilogue drain off,
# 8 unpack tcgen05.st off, 16 weight bulk copies off.
cd "$(dirname "$0")/.."
MASKS=${MASKS:-"0 1 2 4 8 9 16 17 6 22 31"}
if [ "$1" = build ]; then
  for m in $MASKS; do
    QS_NVCC_EXTRA="-DQS_AB=$m" QS_BUILD_DIR=scratch/ab$m/obj QS_LIB_OUT=scratch/ab$m/libqspec_b200.so \
      python paper_2410_11305_b200/build.py > /dev/null || exit 1
  done
  exit 0
fi
mkdir -p gpurun_out
T=${TAG:-ab}
for m in $MASKS; do
  echo "== QS_AB=$m"
  QSPEC_LIB=scratch/ab$m/libqspec_b200.so timeout 300 python scripts/linear_bench.py \
    --shapes ${SHAPES:-28672x8192,12288x4096} --ms ${MS:-1,16,64} --reps 20 2>&1 | \
    python -c "
import json,sys
for l in sys.stdin:
    try: r=json.loads(l)
    except Exception: print(l.rstrip()); continue
    print(f\"{r['shape']:>11} M={r['M']:>3} {r['mode']}: lin {r['us_linear_only']:8.2f} us {r['GBps_linear_only']:7.1f} GB/s | pack+lin {r['us']:8.2f}\")
"
done 2>&1 | tee gpurun_out/${T}.txt

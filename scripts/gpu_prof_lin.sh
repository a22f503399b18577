#!/bin/bash
# ncu --set full of one prepacked linear launch (scripts/prof_linear.py); args via env.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T=${TAG:-pl}
for spec in ${SPECS:-"28672x8192 64 w4a16"}; do :; done
IFS=';' read -ra ALL <<< "${SPECS:-28672x8192 64 w4a16}"
i=0
for spec in "${ALL[@]}"; do
  ncu --set full --import-source on -k regex:linear_tc --launch-skip 2 -c 1 --clock-control none \
    -o gpurun_out/${T}_$i python scripts/prof_linear.py $spec > gpurun_out/${T}_$i.log 2>&1; echo "ncu $spec rc=$?"
  i=$((i+1))
done

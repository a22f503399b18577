#!/bin/bash
# ncu --set full of in-forward linear launches: 4 chain-of-1 launches (QS_CHAIN_SPLIT=1) vs the
# same 4 single launches (QS_EMIT=3), third forward.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T=${TAG:-pf}
QS_EMIT=7 QS_CHAIN_SPLIT=1 timeout 600 ncu --set full --import-source on -k regex:linear_chain --launch-skip 8 -c 4 --clock-control none \
  -o gpurun_out/${T}_chain python scripts/prof_forward.py 16 low 3 > gpurun_out/${T}_chain.log 2>&1; echo "chain rc=$?"
QS_EMIT=3 timeout 600 ncu --set full --import-source on -k regex:linear_tc --launch-skip 19 -c 4 --clock-control none \
  -o gpurun_out/${T}_single python scripts/prof_forward.py 16 low 3 > gpurun_out/${T}_single.log 2>&1; echo "single rc=$?"
tail -n 3 gpurun_out/${T}_chain.log; tail -n 3 gpurun_out/${T}_single.log

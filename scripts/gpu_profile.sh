# ncu evidence for profiles/: launch lists + one --set full capture per hot kernel (1 GPU).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T=${TAG:-p}
ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_b16.csv python scripts/profile_step.py --batch 16 > /dev/null 2>&1; echo "l16 $?"
ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_ar1.csv python scripts/profile_step.py --batch 1 --algorithm greedy > /dev/null 2>&1; echo "l1 $?"
# dominant kernel, full set: verify gate_up (B=16, T=64, L=3) and draft gate_up (T=16, L=1)
ncu --set full --import-source on --nvtx --nvtx-include "step/" -k regex:linear_tc -s 389 -c 1 --clock-control none -o gpurun_out/${T}_verify_gateup python scripts/profile_step.py --batch 16 > /dev/null 2>&1; echo "f1 $?"
ncu --set full --import-source on --nvtx --nvtx-include "step/" -k regex:linear_tc -s 2 -c 1 --clock-control none -o gpurun_out/${T}_draft_gateup python scripts/profile_step.py --batch 16 > /dev/null 2>&1; echo "f2 $?"
ncu --set full --import-source on --nvtx --nvtx-include "step/" -k regex:attn -s 1 -c 1 --clock-control none -o gpurun_out/${T}_attn python scripts/profile_step.py --batch 16 > /dev/null 2>&1; echo "f3 $?"
ncu --set full --import-source on --nvtx --nvtx-include "step/" -k regex:act_pack -s 2 -c 1 --clock-control none -o gpurun_out/${T}_pack python scripts/profile_step.py --batch 16 > /dev/null 2>&1; echo "f4 $?"

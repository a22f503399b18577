# Full round evidence on one B200: gpu tests, smoke, bench (both arms), ncu launch list + full captures.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T=${TAG:-r}
nvidia-smi > gpurun_out/${T}_smi.txt 2>&1
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/${T}_tests.log 2>&1; echo "tests rc=$?" | tee -a gpurun_out/${T}_rc.txt; tail -3 gpurun_out/${T}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?" | tee -a gpurun_out/${T}_rc.txt
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?" | tee -a gpurun_out/${T}_rc.txt
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${T}_bench_ref.json 2> gpurun_out/${T}_bench_ref.err; echo "ref rc=$?" | tee -a gpurun_out/${T}_rc.txt
timeout 600 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_b16.csv python scripts/profile_step.py --batch 16 > gpurun_out/${T}_ncu1.log 2>&1; echo "ncu1 rc=$?" | tee -a gpurun_out/${T}_rc.txt
timeout 600 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_ar1.csv python scripts/profile_step.py --batch 1 --algorithm greedy > gpurun_out/${T}_ncu2.log 2>&1; echo "ncu2 rc=$?" | tee -a gpurun_out/${T}_rc.txt
timeout 600 ncu --set full --import-source on --nvtx --nvtx-include "step/" -k regex:linear_tc -s 389 -c 1 --clock-control none -o gpurun_out/${T}_verify_gateup python scripts/profile_step.py --batch 16 > gpurun_out/${T}_ncu3.log 2>&1; echo "ncu3 rc=$?" | tee -a gpurun_out/${T}_rc.txt
timeout 600 ncu --set full --import-source on --nvtx --nvtx-include "step/" -k regex:linear_tc -s 2 -c 1 --clock-control none -o gpurun_out/${T}_draft_gateup python scripts/profile_step.py --batch 16 > gpurun_out/${T}_ncu4.log 2>&1; echo "ncu4 rc=$?" | tee -a gpurun_out/${T}_rc.txt
timeout 600 ncu --set full --import-source on --nvtx --nvtx-include "step/" -k regex:attn -s 1 -c 1 --clock-control none -o gpurun_out/${T}_attn python scripts/profile_step.py --batch 16 > gpurun_out/${T}_ncu5.log 2>&1; echo "ncu5 rc=$?" | tee -a gpurun_out/${T}_rc.txt
cat gpurun_out/${T}_bench.json

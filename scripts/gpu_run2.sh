cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/r2_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2_rc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2_rc.txt
timeout 900 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo "bench rc=$?" >> gpurun_out/r2_rc.txt
timeout 600 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches.csv python scripts/profile_step.py --batch 16 > gpurun_out/r2_ncu1.log 2>&1; echo "ncu1 rc=$?" >> gpurun_out/r2_rc.txt
timeout 600 ncu --set full --import-source on --nvtx --nvtx-include "step/" -k regex:linear_tc -s 389 -c 1 --clock-control none -o gpurun_out/r2_verify_gateup python scripts/profile_step.py --batch 16 > gpurun_out/r2_ncu2.log 2>&1; echo "ncu2 rc=$?" >> gpurun_out/r2_rc.txt
timeout 600 ncu --set full --import-source on --nvtx --nvtx-include "step/" -k regex:linear_tc -s 2 -c 1 --clock-control none -o gpurun_out/r2_draft_gateup python scripts/profile_step.py --batch 16 > gpurun_out/r2_ncu3.log 2>&1; echo "ncu3 rc=$?" >> gpurun_out/r2_rc.txt
cat gpurun_out/r2_rc.txt

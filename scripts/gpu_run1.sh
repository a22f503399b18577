cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "act_quant or random_init or library" > gpurun_out/t1.log 2>&1; echo "t1 rc=$?" >> gpurun_out/rc.txt
timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "integer_core" > gpurun_out/t2.log 2>&1; echo "t2 rc=$?" >> gpurun_out/rc.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "not integer_core and not act_quant and not random_init" > gpurun_out/t3.log 2>&1; echo "t3 rc=$?" >> gpurun_out/rc.txt
tail -5 gpurun_out/t*.log

timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu.log
bash profiles/quick_all.sh 2>&1 | tee gpurun_out/quick_all.txt
bash profiles/ncu_capture.sh r02_minhash_cfg2 minhash_kernel --workload cfg2
bash profiles/ncu_capture.sh r02_lsh_cfg4b lsh_kernel --workload cfg4 --sets 200000

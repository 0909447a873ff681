timeout 900 python -m pytest tests/test_shard.py tests/test_round2.py -m gpu -x -q > gpurun_out/pytest_shard.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_shard.log
timeout 2400 python tests/parity_report.py > gpurun_out/parity.log 2>&1; echo parity rc=$?; tail -12 gpurun_out/parity.log
mkdir -p gpurun_out/profiles_r02 && cp -f profiles/r02/parity_report.json gpurun_out/profiles_r02/ 2>/dev/null
SKIP=6 bash profiles/ncu_capture.sh r02_lsh_cfg4c lsh_kernel --workload cfg4 --sets 200000
bash profiles/ncu_capture.sh r02_minhash_cfg3_k1024 minhash_kernel --workload cfg3 --k 1024 --sets 200000
bash profiles/ncu_capture.sh r02_minhash_cfg5 minhash_kernel --workload cfg5 --sets 1000000

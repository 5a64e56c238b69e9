set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/p_pool.log 2>&1; echo "pytest_exit=$?" >> gpurun_out/p_pool.log
timeout 300 python scripts/lat_kernels.py > gpurun_out/lat_pool.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_pool.log 2>&1
PB_ENC_POOL=0 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_nopool.log 2>&1
echo done

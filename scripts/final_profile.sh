#!/bin/bash
# End-of-round evidence on one B200 (run under gpurun from the repo root):
# GPU tests, the bench line, every config, the launch list of the bench
# command (ncu, cold-cache serialised: compare shares, not absolutes), ncu
# --set full of the step's top kernels, and the NTT sweep kernel.
set -u
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/final_pytest_gpu.log 2>&1; echo "pytest_exit=$?" >> gpurun_out/final_pytest_gpu.log
python bench.py --steps 10 --warmup 3 > gpurun_out/final_bench.log 2>&1; echo "bench_exit=$?" >> gpurun_out/final_bench.log
python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/final_bench_ref.log 2>&1
python scripts/bench_configs.py c1 c2 c3 c4 c5 c2p c3p c4p --cpu > gpurun_out/final_bench_configs.log 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/final_bench_short.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv \
      --log-file gpurun_out/final_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/final_ncu_launch.log 2>&1
python scripts/prof_step.py > gpurun_out/final_p1.log 2>&1 && \
  ncu --set full --clock-control none --import-source on --profile-from-start off \
      -k regex:"k_encrypt_sk|k_mac_pipe|k_decrypt_share_cluster" -c 6 -o gpurun_out/final_prof_step python scripts/prof_step.py > gpurun_out/final_ncu_full.log 2>&1
echo done

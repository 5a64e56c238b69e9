#!/bin/bash
# End-of-round evidence on one B200 (run under gpurun from the repo root):
# GPU tests, the bench line, every config, the launch list of the bench
# command (ncu, cold-cache serialised: compare shares, not absolutes), the
# DRAM traffic of one step's kernels, ncu --set full of the step's top
# kernels, a CUPTI timeline and the step breakdown.
set -u
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/final_pytest_gpu.log 2>&1; echo "pytest_exit=$?" >> gpurun_out/final_pytest_gpu.log
python bench.py --steps 20 --warmup 3 > gpurun_out/final_bench.log 2>&1; echo "bench_exit=$?" >> gpurun_out/final_bench.log
python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/final_bench_ref.log 2>&1
python scripts/bench_configs.py c1 c2 c3 c4 c5 c2p c3p c4p --cpu > gpurun_out/final_bench_configs.log 2>&1
python scripts/step_breakdown.py > gpurun_out/final_step_breakdown.log 2>&1
python scripts/timeline.py mnist_mlp > gpurun_out/final_timeline.log 2>&1
python scripts/prof_step.py > gpurun_out/final_p0.log 2>&1 && \
  ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv --log-file gpurun_out/final_step_traffic.csv python scripts/prof_step.py > gpurun_out/final_ncu_traffic.log 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/final_bench_short.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
      --log-file gpurun_out/final_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/final_ncu_launch.log 2>&1
python scripts/prof_step.py > gpurun_out/final_p1.log 2>&1 && \
  ncu --set full --clock-control none --import-source on --profile-from-start off \
      -k regex:"k_encrypt_sk|k_mac_ws|k_decrypt_share_cluster|k_encode_plain_mont|k_mask_ntt" -c 8 \
      -o gpurun_out/final_prof_step python scripts/prof_step.py > gpurun_out/final_ncu_full.log 2>&1
echo done

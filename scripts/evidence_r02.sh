#!/bin/bash
# Round-2 evidence on one B200 (run under gpurun from the repo root): GPU
# tests, the bench line (+ reference arm), the launch list of the bench
# command (ncu, PB_HANDOFF=0 so no kernel waits on the host; cold-cache,
# serialised: compare shares, not absolutes), the DRAM traffic of one step,
# and ncu --set full of the step's top kernels and of every C5 / round-2
# kernel.  Every ncu command runs only after the same command exited 0.
set -u
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/r02_pytest_gpu.log 2>&1; echo "pytest_exit=$?" >> gpurun_out/r02_pytest_gpu.log
python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo "bench_exit=$?" >> gpurun_out/r02_bench.err
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r02_bench_ref.json 2> gpurun_out/r02_bench_ref.err
python scripts/prof_step.py > gpurun_out/r02_p0.log 2>&1 && \
  ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv --log-file gpurun_out/r02_step_traffic.csv python scripts/prof_step.py > gpurun_out/r02_ncu_traffic.log 2>&1
PB_HANDOFF=0 python bench.py --steps 2 --warmup 3 --no-cpu --no-configs > gpurun_out/r02_bench_short.log 2>&1 && \
  PB_HANDOFF=0 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
      --log-file gpurun_out/r02_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-configs > gpurun_out/r02_ncu_launch.log 2>&1
python scripts/prof_step.py > gpurun_out/r02_p1.log 2>&1 && \
  ncu --set full --clock-control none --import-source on --profile-from-start off \
      -k regex:"k_encrypt_sk|k_enc_noise|k_mac_ws|k_decrypt_share_cluster|k_encode_plain_mont|k_mask_ntt|k_dealer" -c 10 \
      -o gpurun_out/r02_prof_step python scripts/prof_step.py > gpurun_out/r02_ncu_step.log 2>&1
for w in tc nl ntt32k maskmac; do
  python scripts/prof_round2.py $w > gpurun_out/r02_p_$w.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -c 6 -o gpurun_out/r02_prof_$w python scripts/prof_round2.py $w > gpurun_out/r02_ncu_$w.log 2>&1
done
python scripts/prof_mac.py > gpurun_out/r02_p_mac.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_mac" -c 4 -o gpurun_out/r02_prof_mac python scripts/prof_mac.py > gpurun_out/r02_ncu_mac.log 2>&1
python scripts/prof_decrypt.py > gpurun_out/r02_p_dec.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_decrypt" -c 4 -o gpurun_out/r02_prof_dec python scripts/prof_decrypt.py > gpurun_out/r02_ncu_dec.log 2>&1
# summaries on the box (the .ncu-rep files are too large to bring back)
for r in gpurun_out/r02_prof_*.ncu-rep; do
  b=$(basename $r .ncu-rep)
  python scripts/ncu_summary.py $r > gpurun_out/${b}_summary.txt 2>&1
  ncu -i $r --page raw --csv > gpurun_out/${b}_raw.csv 2>/dev/null
  gzip -f gpurun_out/${b}_raw.csv
done
python scripts/ncu_source_lines.py gpurun_out/r02_prof_step.ncu-rep k_encrypt_sk 30 > gpurun_out/r02_enc_source_lines.txt 2>&1
python scripts/ncu_source_lines.py gpurun_out/r02_prof_tc.ncu-rep k_tc_ring_gemm 30 > gpurun_out/r02_tc_source_lines.txt 2>&1
python scripts/ncu_source_lines.py gpurun_out/r02_prof_nl.ncu-rep k_nl 30 > gpurun_out/r02_nl_source_lines.txt 2>&1
rm -f gpurun_out/*.ncu-rep
gzip -f gpurun_out/r02_launches_bench.csv gpurun_out/r02_step_traffic.csv
echo done

# A/B of an env knob on the bench value: bash scripts/ab_bench.sh VAR valA valB [reps]
set -u
VAR=$1; A=$2; B=$3; R=${4:-3}
mkdir -p gpurun_out
for i in $(seq 1 $R); do
  for v in $A $B; do
    env $VAR=$v timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$VAR=$v', round(d['value']), round(d['e2e']['value']), round(d['ms_per_step']*1e3,1))" >> gpurun_out/ab.log
  done
done

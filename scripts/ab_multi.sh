# A/B/C of one env knob on the bench value: bash scripts/ab_multi.sh VAR reps val1 val2 ...
VAR=$1; shift; R=$1; shift
for i in $(seq 1 $R); do for v in "$@"; do
env $VAR=$v timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$VAR=$v', round(d['value']), round(d['e2e']['value']), round(d['ms_per_step']*1e3,1))" >> gpurun_out/ab.log
done; done

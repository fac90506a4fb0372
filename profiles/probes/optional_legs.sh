# Every optional bench leg on the current tree, one process each -> gpurun_out/optional_legs_final.jsonl
# usage (repo root): bash profiles/probes/optional_legs.sh
for spec in "batch8x8:--batch 8x8" "corun:--corun" "crossover:--crossover" "granularity:--granularity" "hash64:--hash 64" "offload:--offload" "pool4:--pool 4" "sensitivity:--sensitivity" "serve32:--serve 32" "sweep:--sweep"; do
  name=${spec%%:*}; flags=${spec#*:}
  t0=$(date +%s)
  timeout 900 python bench.py --steps 20 --warmup 3 --no-e2e --no-stall --no-config3 --no-config5 --no-cpu-baseline $flags 2>gpurun_out/leg_$name.err | tail -1 > gpurun_out/leg_$name.json
  rc=$?; t1=$(date +%s)
  python -c "
import json,sys
try:
    d=json.load(open('gpurun_out/leg_$name.json')); print(json.dumps({'flag':'$name','rc':$rc,'wall_s':$t1-$t0,'legs':d.get('legs',{})}))
except Exception as e:
    print(json.dumps({'flag':'$name','rc':$rc,'error':str(e)}))
" >> gpurun_out/optional_legs_final.jsonl
done
echo done

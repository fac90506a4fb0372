for cps in 2 3 4; do for st in 2 3 4 16; do
OC_BULK_CTAS_PER_SM=$cps OC_BULK_STAGES=$st timeout 120 python bench.py --steps 200 --warmup 10 --no-e2e --no-stall --no-config3 --no-config5 --no-cpu-baseline > gpurun_out/sw.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/sw.json').read().strip().splitlines()[-1]);print(json.dumps({'cps':$cps,'stages':$st,'value':round(d['value'],1),'X0':d['kernel']['X0_us_isolated'],'iso_p50':d['kernel']['isolated_launch_us']['p50']}))" >> gpurun_out/sweep_cfg.txt
done; done

mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu 2>&1 | tail -6
python bench.py > gpurun_out/bench10.json 2> gpurun_out/bench10.err
tail -3 gpurun_out/bench10.err
python -c "
import json; d=json.load(open('gpurun_out/bench10.json'))
print('value', round(d['value']/1e6,2), 'ms', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']/1e6,2), 'cpu', d['cpu_baseline'] and round(d['cpu_baseline']['value']/1e6,3), 'clocks', d['clocks'])
print('roof', d['roofline'])
print('modes', {k: round(v['evals_per_s']/1e6,1) for k,v in d['modes'].items()})
"
timeout 900 python tools/parity_report.py > gpurun_out/parity.log 2>&1; tail -20 gpurun_out/parity.log

# bench.py once, printed as a one-line summary (box-variance sampling)
timeout 400 python bench.py > gpurun_out/bench_var.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/bench_var.json'))
print(json.dumps({'value': d['value'], 'median': d['kernel_us']['median'], 'min': d['kernel_us']['min'],
  'frac': d['roofline']['frac'], 'e2e': d['e2e']['value'], 'weave': d.get('weave_llama70b_tp8_shapes_us'),
  'cpu_ms': round(d['cpu_baseline']['value'] / 1e3, 1), 'clocks': d['clocks']}))"
nvidia-smi --query-gpu=serial --format=csv,noheader

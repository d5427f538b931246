#!/bin/bash
# GPU tests + short bench lines for the three evaluation configs + GA breakdown
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu ${PYTEST_ARGS:-} > gpurun_out/qb_pytest.log 2>&1; tail -1 gpurun_out/qb_pytest.log
for c in syn5k pmed40 syn20k; do
  timeout 600 python bench.py --config $c --no-ga --no-cpu-baseline > gpurun_out/qb_$c.json 2>gpurun_out/qb_$c.err
  python -c "import json,sys; d=json.load(open('gpurun_out/qb_$c.json')); print('$c', 'value %.4g' % d['value'], 'ms/step %.4f' % d['ms_per_step'], 'kernel %.4f' % d['roofline']['avg_kernel_ms'], 'e2e %.4g' % d['e2e']['value'])"
done
python tools/ga_breakdown.py device 30 2>&1 | head -2

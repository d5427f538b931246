#!/bin/bash
# e2e (host-buffer pm_evaluate) A/B over the lead-chunk policy, alternating processes
mkdir -p gpurun_out
for c in ${AB_CONFIGS:-syn20k syn5k}; do for r in 1 2; do for lead in ${LEADS:-0 2 4 8}; do
  echo "lead=$lead $c: $(PMB_H2D_LEAD=$lead timeout 600 python bench.py --config $c --steps 20 --no-ga --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("value %.4g e2e %.4g" % (d["value"], d["e2e"]["value"]))')"
done; done; done > gpurun_out/e2e_ab.log 2>&1
cat gpurun_out/e2e_ab.log

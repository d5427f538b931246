timeout 900 python -m pytest tests -x -q -m gpu -k "parity or edge or capi or cpp" 2>&1 | tail -2
for r in 1 2; do for c in syn5k pmed40 syn20k; do
  echo "$c: $(timeout 600 python bench.py --config $c --steps 20 --no-ga --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("value %.4g e2e %.4g" % (d["value"], d["e2e"]["value"]))')"
done; done

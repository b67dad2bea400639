# A/B of library builds (AB_LIBS) on the C2 bench step and the C4 / C5 configs
S='import json,sys; d=json.loads(sys.stdin.read()); print("c2", round(d["ms_per_step"],1), {k:(round(v["avg_launch_ms"],3)) for k,v in d["kernels"].items()})'
for lib in "" ${AB_LIBS}; do
  echo "== ${lib:-in-tree}"
  CT_LIBRARY=$lib python bench.py --no-cpu-baseline --no-e2e --steps 2 2>/dev/null | tail -1 | python -c "$S"
  CT_LIBRARY=$lib python tools/bench_configs.py --only ${CONFIGS:-c4,c5} 2>/dev/null | grep -v "^{" | python -c "
import sys, json
for line in sys.stdin:
    name, _, js = line.partition(' ')
    d = json.loads(js)
    if name == 'c4': print('c4', {k: {a: round(b, 3) for a, b in v.items()} for k, v in d.items() if isinstance(v, dict)})
    elif name == 'c5': print('c5', round(d['s_per_object_iteration'], 4))
    else: print(name, round(d.get('s_per_iteration', 0), 4))
"
done

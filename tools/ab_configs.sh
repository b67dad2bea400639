for lib in "" ${AB_LIBS}; do
  echo "== ${lib:-in-tree}"
  CT_LIBRARY=$lib python tools/bench_configs.py --only ${CONFIGS:-c1,paper} 2>&1 | grep -v "^{" | python -c "
import sys, json
for line in sys.stdin:
    name, _, js = line.partition(' ')
    d = json.loads(js)
    if name == 'c1': print('c1', round(d['report_wall_time_s'], 4), round(d['sart_run_call_s'], 4))
    elif name == 'paper': print('paper', {k: (round(v['report_wall_time_s'], 4), round(v['sart_run_call_s'], 4)) for k, v in d.items() if isinstance(v, dict) and 'report_wall_time_s' in v})
    else: print(name, js[:300])
"
done

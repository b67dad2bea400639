# A/B of an environment switch (AB_ENV, e.g. CT_GATHER_QUAD) over values AB_VALS on configs
for lib in "" ${AB_LIBS}; do
  for v in ${AB_VALS:-1 0}; do
    echo "== ${lib:-in-tree} ${AB_ENV}=$v"
    env ${AB_ENV}=$v CT_LIBRARY=$lib python tools/bench_configs.py --only ${CONFIGS:-c4,c5} 2>/dev/null | grep -v "^{" | python -c "
import sys, json
for line in sys.stdin:
    name, _, js = line.partition(' ')
    d = json.loads(js)
    if name == 'c4': print('c4', {k: {a: round(b, 3) for a, b in v.items()} for k, v in d.items() if isinstance(v, dict)})
    elif name == 'c5': print('c5', round(d['s_per_object_iteration'], 4))
    else: print(name, round(d.get('s_per_iteration', 0), 4))
"
  done
done

# A/B of BP variants (AB_LIBS) with and without the quad footprints
S='import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], {k:(round(v["avg_launch_ms"],3)) for k,v in d["kernels"].items()})'
for lib in "" ${AB_LIBS}; do
  for q in 1 0; do
    echo "== ${lib:-in-tree} quads=$q"
    CT_BP_QUADS=$q CT_LIBRARY=$lib python bench.py --no-cpu-baseline --no-e2e --steps 2 2>/dev/null | tail -1 | python -c "$S"
  done
done

#!/bin/bash
# A/B of library variants (build_ab/<name>.so, tools/build_variant.sh) on one
# GPU: C5 object-iteration and C2 iteration device times from bench.py, plus
# a parity subset.  usage: tools/ab_run.sh name1 name2 ...
for v in "$@"; do
  echo "== $v"
  CT_LIBRARY=build_ab/$v.so timeout 600 python bench.py --objects 2 --steps 2 --warmup 1 \
      --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json, sys
d = json.loads(sys.stdin.read())
k = d['kernels']
print('C5 s/obj-it %.4f  fp_corr %.2f ms  fp_resid %.2f ms  bp %.2f ms  C2 ms/it %.2f' % (
    d['s_per_object_iteration'], k['fp_correction']['avg_launch_ms'],
    k['fp_residual']['avg_launch_ms'], k['bp_update']['avg_launch_ms'],
    d['c2']['ms_per_iteration']))"
  if [ "${PARITY:-1}" = "1" ]; then
    CT_LIBRARY=build_ab/$v.so timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_fullsize.py \
        tests/test_gpu_projector.py tests/test_gpu_recon.py 2>&1 | tail -1
  fi
done

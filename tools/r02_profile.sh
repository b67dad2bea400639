#!/bin/bash
# Round-2 measurement pass on one B200 (run under gpurun from the repo root):
# the bench, the on-chip peaks microbenchmark, the ncu launch list of the bench
# and one `ncu --set full` capture of each config's SART kernels (tools/prof.py).
# ncu reports stay in /tmp (gpurun copies back <= 64 MiB); their raw-page CSV
# and details text come back under gpurun_out/.
set -u
mkdir -p gpurun_out /tmp/ncu
[ -x tools/microbench/microbench ] || nvcc -gencode arch=compute_100a,code=sm_100a -O3 \
    -o tools/microbench/microbench tools/microbench/microbench.cu
if [ "${MICRO:-1}" = "1" ]; then
  tools/microbench/microbench > gpurun_out/r02_microbench.json 2> gpurun_out/r02_microbench.err
fi
if [ "${BENCH:-1}" = "1" ]; then
  python bench.py ${BENCH_ARGS:-} > gpurun_out/r2_bench.log 2>&1
  echo "bench rc=$?"
fi
if [ "${NCU:-1}" = "1" ]; then
  if [ "${LAUNCHES:-1}" = "1" ]; then
    ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
        --log-file gpurun_out/r2_launches.csv python bench.py --steps 1 --warmup 1 --objects 1 \
        --no-e2e --no-cpu-baseline --no-c2 > gpurun_out/r2_ncu_launch.log 2>&1
    echo "launch list rc=$?"
  fi
  for cfg in ${NCU_CONFIGS:-c5 c2}; do
    ncu --set full --metrics lts__t_bytes.sum,sm__pipe_fma_cycles_active.sum,sm__cycles_active.sum \
        --clock-control none --import-source on --profile-from-start off -f \
        -o /tmp/ncu/r2_ncu_$cfg python tools/prof.py --config $cfg --reps 1 \
        > gpurun_out/r2_ncu_$cfg.log 2>&1
    echo "ncu $cfg rc=$?"
    ncu -i /tmp/ncu/r2_ncu_$cfg.ncu-rep --page raw --csv > gpurun_out/r2_ncu_${cfg}_raw.csv
    ncu -i /tmp/ncu/r2_ncu_$cfg.ncu-rep --page details > gpurun_out/r2_ncu_${cfg}_details.txt
  done
fi
du -sh gpurun_out

#!/bin/bash
# ncu evidence for the round: launch list of a short bench run, dram/tensor metrics of
# the fused kernels at the bench size, and one --set full capture.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
NCU=ncu
echo "== launch list"
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2> gpurun_out/launches.err
tail -2 gpurun_out/launches.err
echo "== metrics c2"
timeout 900 $NCU --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tensor_subpipe_imma.sum,lts__t_bytes.sum,sm__cycles_elapsed.avg.per_second \
  --clock-control none -k regex:tally2 -s 1 -c 1 --csv --log-file gpurun_out/metrics_c2.csv \
  python scripts/profile_step.py --workload c2 --reps 2 > /dev/null 2> gpurun_out/metrics_c2.err
tail -2 gpurun_out/metrics_c2.err
echo "== metrics c4"
timeout 900 $NCU --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum \
  --clock-control none -k regex:tally3 -s 1 -c 1 --csv --log-file gpurun_out/metrics_c4.csv \
  python scripts/profile_step.py --workload c4 --reps 2 > /dev/null 2> gpurun_out/metrics_c4.err
tail -2 gpurun_out/metrics_c4.err
echo "== full c2-small"
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:tally2 -s 1 -c 1 \
  -o gpurun_out/prof_tally2 -f python scripts/profile_step.py --workload c2 --n_v ${FULL_NV:-8192} --reps 2 > /dev/null 2> gpurun_out/full.err
tail -2 gpurun_out/full.err
ls -la gpurun_out

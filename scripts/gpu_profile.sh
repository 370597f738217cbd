#!/bin/bash
# ncu evidence for the round (one GPU; never a multi-rank command), plus plain bench lines.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second
echo "== bench lines (no profiler)"
for wl in c2 c4 c4f32 c4ck c2s c4s c4paper c2pop c2fs; do
  E=--no-e2e; C=--no-cpu; [ $wl = c2 ] && E= && C=
  ST=${STEPS:-5}; [ $wl = c4s ] && ST=1; [ $wl = c4paper ] && ST=1; [ $wl = c4 ] && ST=2; [ $wl = c4f32 ] && ST=2; [ $wl = c4ck ] && ST=2
  timeout 900 python bench.py --workload $wl --steps $ST --warmup 3 $E $C > gpurun_out/bench_$wl.json 2> gpurun_out/bench_$wl.err
  tail -1 gpurun_out/bench_$wl.json | cut -c1-200
done
echo "== launch lists"
for wl in c2 c4 c2pop c2fs c2s c4s c4paper; do
  S=2; [ $wl = c4 ] && S=1; [ $wl = c2pop ] && S=1; [ $wl = c4s ] && S=1; [ $wl = c4paper ] && S=1
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$wl.csv python bench.py --workload $wl --steps $S --warmup 1 --no-e2e --no-cpu > /dev/null 2> gpurun_out/launches_$wl.err
  tail -1 gpurun_out/launches_$wl.err
done
echo "== metrics c2 (pack, expand, tally2) and c4 (tally3 one stage)"
timeout 900 ncu --metrics $M --clock-control none -k regex:"pack|expand|tally2" -s 3 -c 3 --csv \
  --log-file gpurun_out/metrics_c2.csv python scripts/profile_step.py --workload c2 --reps 2 > /dev/null 2>&1
timeout 900 ncu --metrics $M --clock-control none -k regex:tally3 -s 1 -c 1 --csv \
  --log-file gpurun_out/metrics_c4.csv python scripts/profile_step.py --workload c4 --reps 2 > /dev/null 2>&1
echo "== full tally2 c2 / tally3 c4"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:tally2 -s 1 -c 1 \
  -o gpurun_out/full_tally2_c2 -f python scripts/profile_step.py --workload c2 --reps 2 > gpurun_out/full2.log 2>&1
tail -1 gpurun_out/full2.log
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:tally3 -s 1 -c 1 \
  -o gpurun_out/full_tally3_c4 -f python scripts/profile_step.py --workload c4 --reps 2 > gpurun_out/full3.log 2>&1
tail -1 gpurun_out/full3.log
ls -la gpurun_out | tail -30

#!/bin/bash
# ncu evidence for the round (one GPU; never a multi-rank command).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second
echo "== launch list (bench c2, 2 steps after 1 warm-up)"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2> gpurun_out/launches_c2.err
tail -1 gpurun_out/launches_c2.err
echo "== launch list (bench c4)"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_c4.csv python bench.py --workload c4 --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2> gpurun_out/launches_c4.err
tail -1 gpurun_out/launches_c4.err
echo "== metrics c2 (pack, expand, tally2)"
timeout 900 ncu --metrics $M --clock-control none -k regex:"pack|expand|tally2" -s 3 -c 3 --csv \
  --log-file gpurun_out/metrics_c2.csv python scripts/profile_step.py --workload c2 --reps 2 > /dev/null 2>&1
echo "== metrics c4 (tally3 one stage)"
timeout 900 ncu --metrics $M --clock-control none -k regex:tally3 -s 1 -c 1 --csv \
  --log-file gpurun_out/metrics_c4.csv python scripts/profile_step.py --workload c4 --reps 2 > /dev/null 2>&1
echo "== full tally2 c2"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:tally2 -s 1 -c 1 \
  -o gpurun_out/full_tally2_c2 -f python scripts/profile_step.py --workload c2 --reps 2 > gpurun_out/full2.log 2>&1
tail -1 gpurun_out/full2.log
echo "== full tally3 c4"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:tally3 -s 1 -c 1 \
  -o gpurun_out/full_tally3_c4 -f python scripts/profile_step.py --workload c4 --reps 2 > gpurun_out/full3.log 2>&1
tail -1 gpurun_out/full3.log
echo "== bench"
timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/bench_clk.json 2>&1; cat gpurun_out/bench_clk.json | tail -1 | cut -c1-300
python -c "
import json; d=json.loads(open('gpurun_out/bench_clk.json').read().splitlines()[-1]); print(d['clocks'])"
ls -la gpurun_out

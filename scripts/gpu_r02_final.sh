#!/bin/bash
# Round-2 evidence: default bench line + reference arm, workload lines, launch list of the
# default command, ncu --set full of the sparse 3-way kernel.  Outputs in gpurun_out/r02/.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r02
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
echo "== default"; timeout 900 python bench.py > $O/bench_c2_default.json 2> $O/bench_c2_default.err; tail -1 $O/bench_c2_default.err
echo "== reference"; timeout 600 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err; tail -1 $O/bench_reference.err
for wl in ${WLS:-c2s c2fs c2hwe c4f32 c4ck c4paper c2pop c1}; do
  echo "== $wl"; timeout 600 python bench.py --workload $wl --steps 5 --warmup 3 --no-e2e > $O/bench_$wl.json 2> $O/bench_$wl.err; tail -1 $O/bench_$wl.err
done
echo "== launch list"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_default.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > $O/launches_default.out 2>&1; tail -1 $O/launches_default.out
echo "== ncu tally3s"
STAGE=0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:tally3s -c 1 -f -o $O/t3s \
  python scripts/time3s.py > $O/t3s.log 2>&1; tail -2 $O/t3s.log

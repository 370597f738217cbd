#!/bin/bash
# Round-2 final evidence: GPU suite, sanitizers, default bench + reference arm, c3/c5/c4s
# lines, launch lists (our kernels only) of the default command.  Outputs in gpurun_out/r02b/.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r02b
mkdir -p $O
echo "== smoke"; timeout 300 python __graft_entry__.py smoke 2>&1 | tail -2
echo "== tests"; timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --target-processes all --print-limit 20 python scripts/sanitize_small.py > $O/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|sanitize run ok" $O/sanitize_$tool.log | head -3
done
echo "== default"; timeout 900 python bench.py > $O/bench_c2_default.json 2> $O/bench_c2_default.err; tail -1 $O/bench_c2_default.err
echo "== reference"; timeout 600 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
echo "== c4s"; timeout 600 python bench.py --workload c4s --steps 5 --warmup 3 --no-e2e > $O/bench_c4s.json 2> $O/bench_c4s.err
echo "== c3"; timeout 900 python bench.py --workload c3 --steps 3 --warmup 3 --no-e2e > $O/bench_c3.json 2> $O/bench_c3.err; tail -1 $O/bench_c3.err
echo "== c5"; timeout 1500 python bench.py --workload c5 --steps 1 --warmup 3 --no-e2e > $O/bench_c5.json 2> $O/bench_c5.err; tail -1 $O/bench_c5.err
echo "== grid"; timeout 600 python bench.py --grid 1,1,1 --steps 5 --warmup 3 --no-e2e > $O/bench_grid111.json 2> $O/bench_grid111.err
echo "== launch list"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'tally|expand|pack|fs_|popc' -c 300 --csv \
  --log-file $O/launches_default.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > $O/launches_default.out 2>&1
tail -c 300 $O/launches_default.out

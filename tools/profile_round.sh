#!/usr/bin/env bash
# One GPU box, one call: the bench lines, the per-config numbers and the ncu evidence that
# profiles/ summarises for a round.  Everything lands in gpurun_out/<tag>_*:
#
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash tools/profile_round.sh r2'
#
# Each ncu pass runs only after its command exited 0 without ncu (the numbers printed under ncu
# are never bench values).  Summaries: python tools/launch_summary.py / tools/ncu_lines.py.
set -u
TAG=${1:-r2}
O=gpurun_out
mkdir -p $O
B="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e"

python bench.py > $O/${TAG}_bench_default.json 2> $O/${TAG}_bench_default.err
python bench.py --optimizer sgd --no-cpu > $O/${TAG}_bench_sgd.json 2> $O/${TAG}_bench_sgd.err
timeout 900 python tools/bench_configs.py > $O/${TAG}_configs.jsonl 2> $O/${TAG}_configs.err

# launch lists (cold-cache, serialised: shares, not absolute times)
if $B > /dev/null 2>&1; then
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches_adam.csv $B > /dev/null 2>&1
fi
if $B --optimizer sgd > /dev/null 2>&1; then
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches_sgd.csv $B --optimizer sgd > /dev/null 2>&1
fi
# full captures of the dominant kernels (one launch each after the warm-up launches)
ncu --set full --clock-control none --import-source on -k regex:"demo_tc_adam|demo_fix64" -s 6 -c 2 \
    -o $O/${TAG}_tc_adam -f $B > $O/${TAG}_ncu_adam.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"demo_tc_adam|demo_fix64" -s 6 -c 2 \
    -o $O/${TAG}_tc_sgd -f $B --optimizer sgd > $O/${TAG}_ncu_sgd.log 2>&1
for r in tc_adam tc_sgd; do
  [ -f $O/${TAG}_$r.ncu-rep ] && ncu -i $O/${TAG}_$r.ncu-rep --page raw --csv > $O/${TAG}_$r.raw.csv 2>/dev/null
done
ls -la $O

#!/usr/bin/env bash
# Multi-GPU bench lines for profiles/<tag>_scaling.jsonl: every layout of N GPUs given, AdamW and
# SGD (OLMo-2-1B, k=32, sign).  Run on an N-GPU box:
#   /usr/local/graft/bin/gpurun --gpus 4 --timeout 2400 -- 'bash tools/scaling_round.sh r2 4'
TAG=${1:-r2}
N=${2:-4}
O=gpurun_out/${TAG}_scaling_n${N}.jsonl
: > $O
run() {  # layout optimizer extra...
  local lay=$1 opt=$2; shift 2
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29600 \
    bench.py --gpus $N --layout $lay --optimizer $opt --no-cpu "$@" 2>/dev/null | grep '^{' | tail -1 >> $O
}
if [ "$N" = 2 ]; then LAYS="1x2 2x1"; fi
if [ "$N" = 4 ]; then LAYS="1x4 2x2 4x1"; fi
if [ "$N" = 8 ]; then LAYS="1x8 2x4 4x2 8x1"; fi
for lay in $LAYS; do
  run $lay adamw
  run $lay sgd
done
python - "$O" <<'PY'
import json, sys
for l in open(sys.argv[1]):
    d = json.loads(l)
    print(d["config"]["layout"], d["config"]["optimizer"], f'{d["value"] / 1e9:.1f} G params/s', f'{d["ms_per_step"]:.2f} ms',
          "e2e", f'{d["e2e"]["value"] / 1e9:.2f} G' if d.get("e2e") else None)
PY

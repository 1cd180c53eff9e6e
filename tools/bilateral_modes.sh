#!/bin/bash
# Times the bilateral's table-lookup modes (LK_BILATERAL_MODE, see k_bilateral_tile).
# Usage (GPU box): bash tools/bilateral_modes.sh [modes...]
nvidia-smi --query-gpu=serial,clocks.sm,clocks.max.sm,temperature.gpu --format=csv,noheader
for m in ${@:-0 1 2 3}; do
  for rep in 1 2; do
    LK_BILATERAL_MODE=$m python bench.py --steps 40 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.load(sys.stdin); print('mode $m fps', round(d['value']), 'stage9_ms', d['stage_ms']['9'], d['clocks'])"
  done
done

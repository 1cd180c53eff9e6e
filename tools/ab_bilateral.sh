#!/usr/bin/env bash
# A/B of fast-bilateral variants on the KITTI bench (run under gpurun):
#   bash tools/ab_bilateral.sh "LK_BF_TABLE=21 LK_BF_RC=16" "LK_BF_V1=1" ...
mkdir -p gpurun_out
python -m pytest tests/test_gpu_fastpath.py -x -q > gpurun_out/fastpath.log 2>&1; tail -1 gpurun_out/fastpath.log
for cfg in "$@"; do
  env $cfg python bench.py --no-cpu-baseline --steps 30 > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$cfg', round(d['value']), round(d['e2e']['value']), 'bf_ms', round(d['roofline']['kernel_ms'],3), d['stage_ms'])"
done

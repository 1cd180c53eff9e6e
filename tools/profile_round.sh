#!/usr/bin/env bash
# Regenerates the measurement artefacts of a round on a B200 (run under gpurun):
#   bench lines (KITTI batch, hires, reference arm), the per-kernel launch list
#   (gpu__time_duration, cold and serialised) and ncu --set full captures of the
#   two largest kernels. Outputs land in gpurun_out/; summaries are copied to
#   profiles/ by hand (tools/launch_summary.py, tools/ncu_summary.py).
set -u
OUT=${OUT:-gpurun_out}
mkdir -p "$OUT"
python bench.py > "$OUT/bench_kitti.json" 2> "$OUT/bench_kitti.err"
python bench.py --config hires --steps 20 > "$OUT/bench_hires.json" 2> "$OUT/bench_hires.err"
python bench.py --impl reference --steps 3 --warmup 1 > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file "$OUT/launches.csv" python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    > "$OUT/ncu_launches.log" 2>&1
for k in k_bilateral_fast k_sobel_refine; do
    ncu --set full --clock-control none --import-source on -k "regex:$k" -s 2 -c 1 \
        -o "$OUT/${k}_full" -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
        > "$OUT/ncu_${k}.log" 2>&1
done
echo done

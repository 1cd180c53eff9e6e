#!/usr/bin/env bash
# Regenerates the measurement artefacts of a round on a B200 (run under gpurun):
#   bench lines (KITTI batch, hires, stereo pairs, the reference arm), the
#   per-kernel launch list of device-resident replays in the product
#   configuration (gpu__time_duration; cold and serialised by ncu), a single-
#   range launch list with DRAM bytes (tools/traffic_json.py -> profiles/
#   traffic.json), and ncu --set full captures of the front-end kernels, K1 and
#   the vote accumulation. Outputs land in gpurun_out/; summaries are copied to
#   profiles/ (tools/launch_summary.py, tools/ncu_summary.py, tools/ncu_lines.py).
set -u
OUT=${OUT:-gpurun_out}
mkdir -p "$OUT"
python bench.py > "$OUT/bench_kitti.json" 2> "$OUT/bench_kitti.err"
python bench.py --config hires --steps 20 > "$OUT/bench_hires.json" 2> "$OUT/bench_hires.err"
python bench.py --stereo --steps 10 > "$OUT/bench_stereo.json" 2> "$OUT/bench_stereo.err"
python bench.py --impl reference --steps 3 --warmup 1 > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"
# the launch list of the bench command itself (the contract's), and a clean one:
# single-range 256-frame device-resident replays (one launch per kernel per step)
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file "$OUT/launches.csv" python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    > "$OUT/ncu_launches.log" 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -c 200 --csv --log-file "$OUT/launches_single_range.csv" python tools/kernel_times.py kitti 3 \
    > "$OUT/ncu_launches_sr.log" 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -c 200 --csv --log-file "$OUT/launches_hires_single_range.csv" python tools/kernel_times.py hires 3 \
    > "$OUT/ncu_launches_hires.log" 2>&1
for k in ${KERNELS:-k_prescreen k_bilateral_need k_vanish k_energy k_refine_exact k_m0_m1 k_gamma_fit k_sobel_screen k_sobel_decide k_edge_emit_tiles k_vdisparity}; do
    ncu --set full --clock-control none --import-source on -k "regex:$k" -s 2 -c 1 \
        -o "$OUT/${k}_full" -f python tools/kernel_times.py kitti 2 \
        > "$OUT/ncu_${k}.log" 2>&1
    python tools/ncu_summary.py "$OUT/${k}_full.ncu-rep" > "$OUT/${k}_ncu.txt" 2>&1
    python tools/ncu_lines.py "$OUT/${k}_full.ncu-rep" "$k" 25 > "$OUT/${k}_lines.txt" 2>&1
    # the summaries are what is kept; the reports would exceed gpurun's 64 MiB copy-back
    [ -n "${KEEP_REPS:-}" ] || rm -f "$OUT/${k}_full.ncu-rep"
done
python tools/fraction_table.py "$OUT"/k_*_ncu.txt > "$OUT/fractions.md" 2>&1
echo done

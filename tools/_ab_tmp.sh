timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_v.log 2>&1
for L in ab/lib_old.so paper_1807_02752_b200/liblanekit_b200.so; do
  for cfg in kitti hires; do
  LK_LIBRARY=$L timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_vanish" -c 20 --csv --log-file gpurun_out/v.csv python tools/kernel_times.py $cfg 3 > /dev/null 2>&1
  echo "$L $cfg $(python tools/launch_summary.py gpurun_out/v.csv 2>/dev/null | head -1)" >> gpurun_out/v.txt
  done
  LK_LIBRARY=$L python bench.py --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/vb_$(basename $L).json
  LK_LIBRARY=$L python bench.py --no-cpu-baseline --config hires --steps 20 2>/dev/null | tail -1 > gpurun_out/vh_$(basename $L).json
done

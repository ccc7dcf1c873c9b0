# fp32 DRAM bytes vs L2 fetch granularity (tuning; stdout only)
for f in -1 32 64 128; do
  ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:step_kernel -s 3 -c 1 --csv python scripts/step_sweep.py --geometry channel --n 512 --precision f32 --variants full --steps 2 --l2-fetch $f 2>&1 | grep -E "step_kernel|mlups" | sed -E 's/.*"(dram__bytes_[a-z]+.sum|gpu__time_duration.sum)","[a-z]+","([0-9.]+)"/\1 \2/' | sed "s/^/fetch $f: /" | cut -c1-60
  timeout 300 python scripts/step_sweep.py --geometry channel --n 512 --precision f32 --variants full --steps 20 --l2-fetch $f | cut -c 1-50,230-330
done

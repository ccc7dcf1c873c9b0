# fp32 DRAM bytes per node vs domain shape (tuning; stdout only)
for g in "duct_z --n 256 --length 2048" "channel --n 512" "duct_z --n 1024 --length 128" "channel --n 256"; do
  for t in b200 xyz; do
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:step_kernel -s 3 -c 1 --csv python scripts/step_sweep.py --geometry $g --precision f32 --table $t --variants full --steps 2 2>&1 | grep -E "step_kernel|mlups" | sed -E 's/.*"(dram__bytes_[a-z]+.sum|gpu__time_duration.sum)","[a-z]+","([0-9.]+)"/\1 \2/' | sed "s/^/$t $g: /" | cut -c1-200
  done
done

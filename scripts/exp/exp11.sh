# fp32 on 2 M-tile domains: L2 load policy (tuning; stdout only)
for v in base ld1 ld2; do
  if [ $v = base ]; then L=paper_1611_02445_b200/lib/libtlbm.so; else L=build/variants/$v/libtlbm.so; fi
  for g in "channel --n 512" "channel_z --n 1024 --length 128" "channel --n 256"; do
    TLBM_LIB=$L timeout 300 python scripts/step_sweep.py --geometry $g --precision f32 --variants full --steps 20 | sed "s/^/$v /" | cut -c1-60,200-330
  done
  TLBM_LIB=$L timeout 300 python scripts/step_sweep.py --precision f64 --variants full --steps 50 | sed "s/^/$v /" | cut -c1-60,200-330
done
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:step_kernel -s 3 -c 1 --csv python scripts/step_sweep.py --geometry channel --n 512 --precision f32 --variants full --steps 2 2>&1 | grep step_kernel | cut -c 150-400

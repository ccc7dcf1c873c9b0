# A/B on one box: previous commit's library vs current (stdout only)
for r in 1 2; do for v in prev cur; do
  if [ $v = cur ]; then L=paper_1611_02445_b200/lib/libtlbm.so; else L=build/variants/$v/libtlbm.so; fi
  for g in "channel --n 512" "channel --n 256"; do
    TLBM_LIB=$L timeout 300 python scripts/step_sweep.py --geometry $g --precision f64 --variants full --steps 40 --traversal tile 2>/dev/null | sed "s/^/$v /" | cut -c1-34,250-330
  done
done; done

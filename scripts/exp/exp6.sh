mkdir -p gpurun_out/exp6
timeout 600 python -m pytest tests/test_gpu_graph.py -q > gpurun_out/exp6/pytest_graph.txt 2>&1; tail -2 gpurun_out/exp6/pytest_graph.txt
for g in "channel --n 512" "channel_z --n 1024 --length 128" "channel --n 256"; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none \
      -k regex:step_kernel -s 5 -c 1 --csv python scripts/step_sweep.py --geometry $g --precision f32 --variants full --steps 2 2>&1 | grep -E "step_kernel|mlups" | cut -c1-400
done
for v in prop32 prop48 prop40; do
  TLBM_LIB=build/variants/$v/libtlbm.so timeout 300 python scripts/step_sweep.py --precision f32 --variants prop --steps 200 | sed "s/^/$v /"
done
TLBM_LIB=build/variants/tpc1/libtlbm.so timeout 300 python scripts/step_sweep.py --geometry channel_z --n 1024 --length 128 --precision f32 --variants full --steps 20 | sed "s/^/tpc1 /"
TLBM_LIB=build/variants/minb12/libtlbm.so timeout 300 python scripts/step_sweep.py --geometry channel_z --n 1024 --length 128 --precision f32 --variants full --steps 20 | sed "s/^/minb12 /"
timeout 300 python scripts/step_sweep.py --geometry channel --n 512 --precision f32 --variants full --steps 20

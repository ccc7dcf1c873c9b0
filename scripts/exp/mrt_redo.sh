# re-run the MRT parts of the r1d pass (step_sweep's MRT branch was broken in it)
O=gpurun_out/r1d
python scripts/step_sweep.py --variants rw,prop,full,mrt > $O/ladder_f64.jsonl 2>/dev/null
python scripts/step_sweep.py --variants full,mrt --arith fma > $O/ladder_f64_fma.jsonl 2>/dev/null
python scripts/step_sweep.py --variants rw,prop,full,mrt --precision f32 > $O/ladder_f32.jsonl 2>/dev/null
for k in "mrt:" "mrt_fma:--arith fma"; do
  n=${k%%:*}; extra=${k#*:}
  ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 6 -c 1 \
      -o $O/prof_step_$n python scripts/step_sweep.py --variants mrt --steps 2 $extra > /dev/null 2>&1
  ncu -i $O/prof_step_$n.ncu-rep --page details > $O/prof_step_${n}_details.txt 2>&1
  ncu -i $O/prof_step_$n.ncu-rep --page raw --csv > $O/prof_step_${n}_raw.csv 2>&1
  rm -f $O/prof_step_$n.ncu-rep
done
cat $O/ladder_f64.jsonl $O/ladder_f64_fma.jsonl $O/ladder_f32.jsonl | cut -c1-20,250-330
ls $O | grep mrt

O=gpurun_out
for spec in "wide_solve_n128 cholqr2 gram_wide_fused" "wide_multiply_n128 svqb2 gram_wide_fused"; do
  set -- $spec
  ncu --set full --clock-control none --import-source on -k regex:$3 -c 1 -o $O/x_$1 python tools/prof_run.py $2 128 22 1 > /dev/null 2>&1
  ncu -i $O/x_$1.ncu-rep --page raw --csv > $O/x_$1.raw.csv 2>/dev/null
  ncu -i $O/x_$1.ncu-rep --page source --csv > $O/x_$1.source.csv 2>/dev/null
  rm -f $O/x_$1.ncu-rep
done
python tools/ncu_summary_csv.py $O/x_wide_solve_n128.raw.csv $O/x_wide_multiply_n128.raw.csv

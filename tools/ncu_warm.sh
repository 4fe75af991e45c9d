# warm-cache (--cache-control none) counters of mid-frame solver launches
for k in k_lambda k_deltap_apply; do
ncu --cache-control none --clock-control none -k regex:$k --launch-skip 42 --launch-count 3 \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,lts__t_bytes.sum \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep -E "k_lambda|k_deltap|gpu__|dram__|lts__|l1tex__|smsp__|sm__" 
done

# The round's verification on one B200 (run from the repo root via gpurun):
# every committed profile regenerated from the current tree into gpurun_out/.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/v_gputests.log 2>&1; tail -2 gpurun_out/v_gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/v_smoke.log
python bench.py > gpurun_out/v_bench.json 2> gpurun_out/v_bench.err; echo "bench rc=$?"
python bench.py --impl reference > gpurun_out/v_bench_ref.json 2> gpurun_out/v_bench_ref.err; echo "reference arm rc=$?"
python tools/slab_probe.py ocean_1m 10 > gpurun_out/v_slab_probe.txt 2>&1
python tools/criterion3.py 80 > gpurun_out/v_crit3.txt 2>&1; cat gpurun_out/v_crit3.txt
python tools/bench_configs.py > gpurun_out/v_configs.json 2> gpurun_out/v_configs_tables.txt; echo "configs rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/v_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-fast > gpurun_out/v_ncu_l.log 2>&1
echo "launch list rc=$?"
for build in parity fast; do
  flag=""; [ $build = fast ] && flag="--fast"
  for k in k_lambda k_deltap_apply; do
    ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 60 --launch-count 1 \
        -o gpurun_out/prof_${k}_${build} -f python tools/prof_kernels.py $flag > gpurun_out/ncu_${k}_${build}.log 2>&1
  done
done
ncu --set full --clock-control none --import-source on -k regex:k_build_lists --launch-skip 6 --launch-count 1 \
    -o gpurun_out/prof_k_build_lists_parity -f python tools/prof_kernels.py > gpurun_out/ncu_build_lists.log 2>&1
echo "full captures rc=$?"

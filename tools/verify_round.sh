set -x
python -m pytest tests -m gpu -q > gpurun_out/v_gputests.log 2>&1; tail -3 gpurun_out/v_gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v_smoke.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/v_smoke.log
python bench.py > gpurun_out/v_bench.json 2> gpurun_out/v_bench.err; echo bench rc=$?
python bench.py --impl reference > gpurun_out/v_bench_ref.json 2> gpurun_out/v_bench_ref.err; echo ref rc=$?
python tools/slab_probe.py ocean_1m 10 > gpurun_out/v_slab_probe.txt 2>&1
python tools/criterion3.py 80 > gpurun_out/v_crit3.txt 2>&1; cat gpurun_out/v_crit3.txt
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/v_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-fast > gpurun_out/v_ncu_l.log 2>&1; echo ncu rc=$?

# One profiling pass on a GPU box (run from the repo root via gpurun):
#  1. the bench line (no profiler),
#  2. the ncu launch list of a short bench run (per-kernel shares),
#  3. ncu --set full of one full-activity launch of the top kernels, parity
#     and fast builds (tools/prof_kernels.py fixes the launch sequence).
set -x
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err || exit 1
cat gpurun_out/bench_n1.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-fast > gpurun_out/ncu_l.log 2>&1
for build in parity fast; do
  flag=""; [ $build = fast ] && flag="--fast"
  for k in k_lambda k_deltap_apply; do
    ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 60 --launch-count 1 \
        -o gpurun_out/prof_${k}_${build} -f python tools/prof_kernels.py $flag > gpurun_out/ncu_${k}_${build}.log 2>&1
  done
done
ncu --set full --clock-control none --import-source on -k regex:k_build_lists --launch-skip 6 --launch-count 1 \
    -o gpurun_out/prof_k_build_lists_parity -f python tools/prof_kernels.py > gpurun_out/ncu_build_lists.log 2>&1
ls -la gpurun_out

# One round-end measurement pass (run under gpurun, one GPU): the default
# bench line, the ncu launch list of a short bench run, and ncu --set full
# captures of the step's dominant kernels on the current build.
#   bash tools/gpu_round.sh <tag>      -> gpurun_out/<tag>_*.{log,csv}, prof_*_<tag>.ncu-rep
TAG=${1:-rXX}
NCU="ncu --set full --import-source on --clock-control none -c 1"
python bench.py > gpurun_out/${TAG}_bench.log 2>&1; echo bench=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/${TAG}_ncu_bench.log 2>&1; echo launches=$?
$NCU -k regex:sim_kernel -o gpurun_out/prof_scls_${TAG} python tools/probe.py one scls 4096 > /dev/null 2>&1; echo scls=$?
$NCU -k regex:dp_mono -o gpurun_out/prof_dp_${TAG} python tools/probe_c3_once.py > /dev/null 2>&1; echo dp=$?
tail -1 gpurun_out/${TAG}_bench.log
$NCU -k regex:sim_sls_merge -o gpurun_out/prof_slsm_${TAG} python tools/probe.py one sls 4096 > /dev/null 2>&1; echo slsm=$?

# ncu captures behind profiles/ncu_summary.json (run under gpurun, one GPU):
#   bash tools/gpu_profile.sh   -> gpurun_out/prof_*_r02b.ncu-rep, r02b_*.log
# then: python tools/summarize_ncu.py report gpurun_out/<rep> <kernel-substring>=<name>
set -x
NCU="ncu --set full --import-source on --clock-control none -c 1"
$NCU -k regex:sim_ils_indep -o gpurun_out/prof_ils_r02b python tools/probe.py one ils 4096 > gpurun_out/r02b_ils.log 2>&1
$NCU -k regex:sim_sls_indep -o gpurun_out/prof_sls_r02b python tools/probe.py one sls 4096 > gpurun_out/r02b_sls.log 2>&1
$NCU -k regex:dp_mono -o gpurun_out/prof_dp_r02b python tools/probe_c3_once.py > gpurun_out/r02b_dp.log 2>&1
$NCU -k regex:gen_kernel -o gpurun_out/prof_gen_r02b python tools/probe.py one sls 4096 > gpurun_out/r02b_gen.log 2>&1
SCLS_B200_LIB=build/prof/libscls_b200.so python tools/probe.py scls-prof 4096 10,15,20,25 > gpurun_out/r02b_sclsprof_sweep.log 2>&1
SCLS_B200_LIB=build/prof/libscls_b200.so python tools/probe.py scls-prof 1 25 > gpurun_out/r02b_sclsprof_one.log 2>&1
python tools/probe.py sweep > gpurun_out/r02b_sweep.log 2>&1

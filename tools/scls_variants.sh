# Build-and-time sweep of the SCLS simulator kernel's occupancy knobs:
#   bash tools/scls_variants.sh "minblocks smem" ...
set -e
for v in "$@"; do
  set -- $v
  touch paper_2406_13511_b200/csrc/sim.cu
  make -C paper_2406_13511_b200/csrc EXTRA="-DSCLS_SIM_MINB=$1 -DSCLS_SPLIT_SMEM=$2" >/dev/null 2>&1
  echo "minb=$1 smem=$2 $(grep -A3 'sim_kernelILi0ELb0ELb0E' build/obj/sim.o.ptxas.txt | sed -n 3p)"
  python tools/probe_sim_policy.py 4096 scls 2 2>&1 | tail -1
done

# Build-and-time sweep of the lean ILS kernel's occupancy knob:
#   bash tools/ils_variants.sh minblocks...
set -e
for v in "$@"; do
  touch paper_2406_13511_b200/csrc/sim.cu
  make -C paper_2406_13511_b200/csrc EXTRA="-DSCLS_ILS_MINB=$v" >/dev/null 2>&1
  echo "minb=$v $(grep -A3 'sim_ils_lean' build/obj/sim.o.ptxas.txt | sed -n 3p)"
  python tools/probe_sim_policy.py 4096 ils 2 2>&1 | tail -1
  python tools/probe_ils_single.py ils 148
done

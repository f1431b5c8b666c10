#!/bin/bash
# Build a variant of the library with extra nvcc defines into build/var_<name>/
#   tools/build_variant.sh <name> "-DSCLS_SPLIT_SMEM=64 ..."
# Use it with SCLS_B200_LIB=build/var_<name>/libscls_b200.so (tools/probe.py).
set -e
HERE=$(cd "$(dirname "$0")/.." && pwd)
make -s -C "$HERE/paper_2406_13511_b200/csrc" -j8 EXTRA="$2" OUT="$HERE/build/var_$1/libscls_b200.so" \
  OBJDIR="$HERE/build/var_$1/obj" > "$HERE/build/var_$1.log" 2>&1 || { tail -20 "$HERE/build/var_$1.log"; exit 1; }
grep -A2 "sim_kernelILi0ELb0ELb0ELi1E" "$HERE/build/var_$1/obj/sim.o.ptxas.txt" | grep -E "stack|registers" | tr '\n' ' '
echo

#!/bin/bash
# Build an experimental liboserve_gpu.so variant into build/<name>/ with extra
# nvcc -D flags (e.g. -DOSERVE_K1_MINB_1=6); load it with OSERVE_GPU_LIB=...
# Usage: scripts/build_variant.sh <name> [nvcc flags...]
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
CS=$ROOT/paper_2602_12151_b200/csrc
name=$1; shift
out=$ROOT/build/$name
mkdir -p "$out"
make -s -C "$CS" >/dev/null
NV=/usr/local/cuda/bin/nvcc
ARCH="-gencode arch=compute_100a,code=sm_100a"
$NV $ARCH -O3 -lineinfo -std=c++17 -ccbin /usr/bin/g++ -Xcompiler -fPIC,-ffp-contract=off -Xptxas -v \
    --expt-relaxed-constexpr -I"$CS" "$@" -c "${SRC:-$CS/oserve_kernels.cu}" -o "$out/oserve_kernels.o" 2> "$out/ptxas.log"
$NV $ARCH -shared -ccbin /usr/bin/g++ -o "$out/liboserve_gpu.so" "$out/oserve_kernels.o" "$CS/oserve_flow.o" \
    "$CS/oserve_aux.o" "$CS/oserve_host.o" -lcudart -ldl
grep -A2 "k_plan_evalILi32ELi[124]ELb1ELi0" "$out/ptxas.log" | grep -E "registers|spill" | tr '\n' ' '; echo

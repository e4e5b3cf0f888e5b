#!/bin/bash
# SASS + ptxas resource usage of one specialization, compiled here (no GPU):
#   tools/sass_of.sh N float|double [stream] [extra nvcc -D flags...]
# writes /tmp/sass/k_N_T[_s].{cubin,sass} and prints the ptxas line.
set -e -o pipefail
N=$1; T=$2; shift 2
K=k_update; SUF=""
if [ "$1" = "stream" ]; then K=k_update_stream; SUF=_s; shift; fi
ROOT=$(cd "$(dirname "$0")/.." && pwd)
D=/tmp/sass; mkdir -p $D
DT=$([ "$T" = double ] && echo 1 || echo 0)
if [ "$K" = k_update ]; then
  cat > $D/entry.cpp <<EOT
#include "jm_plan.h"
#include <cstdio>
int main() { printf("%s", jm::use_mb1($N, $DT) ? "_mb1" : jm::use_rc($N, $DT) ? "_rc" : ""); }
EOT
  g++ -std=c++17 -I $ROOT/paper_1904_08555_b200/csrc/kernels -o $D/entry $D/entry.cpp "$@" && K=$K$($D/entry)
fi
cat > $D/inst.cu <<EOT
#include "jm_plan.h"
#include "jm_update.cuh"
namespace jm {
template __global__ void $K<$N, $T, Addend::Ones, tile_for($N, $DT)>(const $T *, $T *, long long, int);
}
EOT
MB1=""
nvcc -gencode arch=compute_100a,code=sm_100a -cubin -O3 -std=c++17 -lineinfo -Xptxas -v "$@" \
  -I $ROOT/paper_1904_08555_b200/csrc/kernels -o $D/k_${N}_${T}${SUF}.cubin $D/inst.cu 2>&1 | grep -E "registers|spill" | head -4
cuobjdump -sass $D/k_${N}_${T}${SUF}.cubin > $D/k_${N}_${T}${SUF}.sass
echo "$D/k_${N}_${T}${SUF}.sass: $(grep -c '^        /\*[0-9a-f]*\*/' $D/k_${N}_${T}${SUF}.sass) instructions"

#!/bin/bash
# Build a variant library paper_2203_04071_b200/libaxq_$1.so: one translation unit ($2, e.g.
# mm_p4) recompiled with extra nvcc flags ($3..., e.g. -DP4W_IDP_QUADS=3), linked with the
# in-tree objects of the others (run the normal build first).  For same-box A/B via AXQ_LIB.
set -e
NAME=$1; TU=$2; shift 2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
P=$ROOT/paper_2203_04071_b200
NV=/usr/local/cuda/bin/nvcc
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I $ROOT/include"
$NV $FL "$@" -c $P/csrc/$TU.cu -o $P/build/${TU}_$NAME.o
OBJS=$(ls $P/build/*.o | grep -v "_[a-z0-9]*\.o$" | grep -v "/$TU.o$" || true)
OBJS=$(for f in $P/build/*.o; do b=$(basename $f .o); case " axq_api mm_delta8 mm_i16 mm_i32 mm_p4 mm_lstm mm_gconv mm_wide mm_ste " in *" $b "*) [ "$b" != "$TU" ] && echo $f;; esac; done)
$NV -gencode arch=compute_100a,code=sm_100a -shared $OBJS $P/build/${TU}_$NAME.o -o $P/libaxq_$NAME.so
echo "built $P/libaxq_$NAME.so"

#!/bin/bash
# Quick variant for A/B runs of the headline kernels: recompile only the
# fp64 n_t=2 instantiation units (plus tmg_api) from the working tree with extra
# flags, link them with the default build's other objects.
#   bash scripts/ab_quick.sh NAME [extra nvcc flags]   -> build/NAME/libtimemg_b200.so
NAME=$1; shift
SRC=${TMG_OBJDIR:-/tmp/tmg_b200_obj}
OBJ=/tmp/tmg_obj_$NAME
mkdir -p build/$NAME $OBJ
cp -u $SRC/*.o $OBJ/
C=paper_1409_5254_b200/csrc
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC -diag-suppress 1886,128 -I include -I $C"
pids=()
for part in 0 1 2 3; do
  nvcc $FLAGS "$@" -c -DTMG_T=double -DTMG_NT=2 -DTMG_PART=$part -o $OBJ/tmg_inst_f64_2_p$part.o $C/tmg_inst.cu & pids+=($!)
done
nvcc $FLAGS "$@" -c -DTMG_T=double -DTMG_NT=2 -o $OBJ/tmg_inst_f64_2_tail.o $C/tmg_inst_tail.cu & pids+=($!)
nvcc $FLAGS "$@" -c -o $OBJ/tmg_api.o $C/tmg_api.cu & pids+=($!)
rc=0; for p in "${pids[@]}"; do wait $p || rc=1; done
[ $rc = 0 ] || { echo "compile failed"; exit 1; }
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/$NAME/libtimemg_b200.so $OBJ/*.o && echo "built build/$NAME/libtimemg_b200.so"

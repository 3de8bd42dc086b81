#!/bin/bash
# Build a variant of the library into build/<name>/libtimemg_b200.so with extra
# nvcc flags (in-tree, git-ignored, travels to the GPU box); select it at run
# time with TMG_LIB=build/<name>/libtimemg_b200.so.
#   bash scripts/ab_build.sh stage64 -DTMG_STAGE_SLABS_P2=64
NAME=$1; shift
mkdir -p build/$NAME
TMG_LIB=$PWD/build/$NAME/libtimemg_b200.so TMG_OBJDIR=/tmp/tmg_obj_$NAME TMG_NVCC_EXTRA="$*" \
    python -c "from paper_1409_5254_b200 import _native; _native.build(force=True)"

#!/bin/bash
# Build a variant of libstarplat_b200.so with extra -D flags into build/variants/NAME/.
# usage: bash tools/build_variant.sh NAME "-DFOO=1 -DBAR=2"   then  SP_LIB=build/variants/NAME/libstarplat_b200.so
NAME=$1; DEFS=$2
D=build/variants/$NAME; mkdir -p $D/obj
make -s -j8 -C paper_2305_03317_b200/csrc OBJDIR=../../$D/obj LIB=../../$D/libstarplat_b200.so \
    NVFLAGS_EXTRA="$DEFS" > $D/build.log 2>&1 || { tail -20 $D/build.log; exit 1; }
echo "$D/libstarplat_b200.so"

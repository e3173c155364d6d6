#!/bin/bash
# build an A/B variant of the library: build_variant.sh NAME "EXTRA_NVFLAGS"
# -> paper_1607_03399_b200/_variants/NAME/libprismdg_b200.so (load with PDG_LIB_PATH)
set -e
cd "$(dirname "$0")/../paper_1607_03399_b200/csrc"
make -s -j"$(nproc)" OUT="../_variants/$1" EXTRA_NVFLAGS="$2" "../_variants/$1/libprismdg_b200.so"

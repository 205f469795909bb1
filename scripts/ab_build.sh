#!/bin/bash
# Build A/B variants of libaps with extra nvcc flags (compile-time switches only):
#   bash scripts/ab_build.sh NAME "-DFLAG=.. -DFLAG2=.."   ->  paper_1911_08907_b200/libaps_NAME.so
APS_BUILD_OUT=paper_1911_08907_b200/libaps_$1.so APS_NVCC_EXTRA="$2" python -m paper_1911_08907_b200.build

#!/bin/bash
# build an experimental variant of libgi.so: tools/ab_build.sh NAME "-DMACRO=VAL ..."
# -> paper_1805_00923_b200/libgi_NAME.so (load it with GI_LIBGI=...)
cd "$(dirname "$0")/.." || exit 1
GI_BUILD_DIR=paper_1805_00923_b200/_build_$1 GI_BUILD_LIB=paper_1805_00923_b200/libgi_$1.so GI_BUILD_DEFS="$2" \
  python -m paper_1805_00923_b200.build --force > /dev/null && echo "built $1: $2"

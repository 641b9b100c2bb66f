#!/bin/bash
# Build an experimental variant of the product library from a patched copy of
# csrc (never touching the product sources):
#   tools/build_variant.sh NAME PATCH.py [make args...]
# PATCH.py is run inside the copied csrc directory (edits files in place);
# the result lands in paper_2108_13976_b200/lib/variants/NAME/libwdg_b200.so
# (select it with WDG_LIB_VARIANT=NAME; tools only).
set -e
NAME=$1; PATCH=$2; shift 2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
W=/tmp/wdg_variant_$NAME
rm -rf $W && mkdir -p $W/pkg && cp -r $ROOT/paper_2108_13976_b200/csrc $W/pkg/ && cp -r $ROOT/include $W/
rm -rf $W/pkg/lib
if [ -n "$PATCH" ]; then (cd $W/pkg/csrc && python3 $(cd "$(dirname "$PATCH")" && pwd)/$(basename "$PATCH")); fi
make -C $W/pkg/csrc -j8 "$@" > $W/build.log 2>&1 || { tail -30 $W/build.log; exit 1; }
mkdir -p $ROOT/paper_2108_13976_b200/lib/variants/$NAME
cp $W/pkg/lib/libwdg_b200.so $ROOT/paper_2108_13976_b200/lib/variants/$NAME/
grep -A2 "tag_env_kernelILb0ELb1ELb1ELi5ELb1ELb0" $W/pkg/lib/obj/ptxas.log | grep -E "Used|spill" || true
echo "built variant $NAME"

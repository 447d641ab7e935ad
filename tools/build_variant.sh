#!/bin/bash
# Build a tuning variant of liblowdiff (not product): tools/build_variant.sh NAME "-DFLAG ..."
# -> tools/variants/NAME/liblowdiff.so (select it with LOWDIFF_LIB=...)
set -e
NAME=$1; FLAGS=$2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
W=/tmp/ldvar_$NAME
rm -rf $W; mkdir -p $W/pkg $W/include
cp -r $ROOT/paper_2509_04084_b200/csrc $W/pkg/csrc; rm -rf $W/pkg/csrc/build
cp $ROOT/include/*.h $W/include/
mkdir -p $ROOT/tools/variants/$NAME
make -s -C $W/pkg/csrc -j8 EXTRA="$FLAGS" OUT=$ROOT/tools/variants/$NAME/liblowdiff.so > /dev/null
echo built $ROOT/tools/variants/$NAME/liblowdiff.so

#!/bin/bash
# development: build a copy of the package with extra nvcc defines, for A/B
# timing on the GPU box:  tools/build_variant.sh NAME "-DTC_F16_STAGES=4 ..."
# -> variants/NAME/paper_2601_08082_b200 (git-ignored; travels with gpurun)
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; shift
DEST=$ROOT/variants/$NAME/paper_2601_08082_b200
rm -rf "$ROOT/variants/$NAME"; mkdir -p "$DEST"; ln -s "$ROOT/include" "$ROOT/variants/$NAME/include"
cp "$ROOT"/paper_2601_08082_b200/*.py "$DEST/"
cp -r "$ROOT/paper_2601_08082_b200/csrc" "$DEST/csrc"
rm -rf "$DEST/csrc/build"
make -C "$DEST/csrc" -j8 "NVFLAGS=-gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr -I$DEST/csrc/ -I$ROOT/include $*" "$DEST/libtreechol_b200.so" > /dev/null
echo "built $DEST"

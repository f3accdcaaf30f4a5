#!/bin/bash
# Build an A/B variant of libmrf_cuda.so with extra nvcc flags into _variants/
# (git-ignored, travels to the GPU box; select it with MRF_LIB_PATH).
#   bash tools/build_variant.sh <name> "<extra nvcc flags>"
set -e
name=$1; extra=$2
src=$(cd "$(dirname "$0")/.." && pwd)
dst=/tmp/mrf_variant_$name
rm -rf $dst && mkdir -p $dst
cp -r $src/paper_1910_10892_b200 $src/include $dst/
rm -f $dst/paper_1910_10892_b200/libmrf_cuda.so
(cd $dst && MRF_NVCC_EXTRA="$extra" python -c "from paper_1910_10892_b200 import build as B; B.build(force=True)")
mkdir -p $src/_variants
cp $dst/paper_1910_10892_b200/libmrf_cuda.so $src/_variants/libmrf_cuda_$name.so
echo built $src/_variants/libmrf_cuda_$name.so

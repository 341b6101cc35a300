# build a library variant with extra -D flags into build_variants/<name>.so
# usage: bash tools/build_variant.sh <name> [-DFLAG=V ...]   (A/B with tools/gpu_variants.sh)
set -e
name=$1; shift
mkdir -p build_variants
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --fmad=false \
  -Xcompiler -fPIC -shared -I include "$@" paper_2306_01369_b200/csrc/gg_abi.cu -o build_variants/$name.so
echo "built build_variants/$name.so $*"

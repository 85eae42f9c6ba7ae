# developer A/B: libmux_<name>.so = the production objects with prefill.cu rebuilt under extra flags
# usage: bash scripts/build_variant.sh <name> "-DFOO=1 -DBAR"
set -e
cd "$(dirname "$0")/../paper_2504_14489_b200"
NAME=$1; shift
EXTRA="$*"
NVCC=${NVCC:-/usr/local/cuda/bin/nvcc}
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC,-fvisibility=hidden -I ../include"
mkdir -p build_$NAME
$NVCC $FL $EXTRA -DMUX_EXTRA_FLAGS="\"$EXTRA\"" -c csrc/prefill.cu -o build_$NAME/prefill.cu.o
$NVCC $FL $EXTRA -DMUX_EXTRA_FLAGS="\"$EXTRA\"" -c csrc/common.cu -o build_$NAME/common.cu.o
OBJS=$(ls build/*.o | grep -v -e prefill.cu.o -e common.cu.o)
$NVCC -gencode arch=compute_100a,code=sm_100a -shared -o libmux_$NAME.so build_$NAME/prefill.cu.o build_$NAME/common.cu.o $OBJS -cudart static -Xcompiler -fPIC
echo built libmux_$NAME.so

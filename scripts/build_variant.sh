# Build an A/B variant of libfcpb.so into dbg/ with extra -D flags.
#   bash scripts/build_variant.sh NAME "-DFOO=1 -DBAR=2"
NAME=$1; shift
mkdir -p dbg
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -cudart static --expt-relaxed-constexpr $* \
  -shared -o dbg/libfcpb_${NAME}.so paper_2605_08524_b200/csrc/fcpb_api.cu

# Builds libfcpb.so (sm_100a only) in-tree; the .so travels to the GPU box via gpurun.
NVCC ?= /usr/local/cuda/bin/nvcc
SRC_DIR := paper_2605_08524_b200/csrc
LIB := paper_2605_08524_b200/libfcpb.so
SRCS := $(SRC_DIR)/fcpb_api.cu
DEPS := $(wildcard $(SRC_DIR)/*.cuh $(SRC_DIR)/*.h) include/fcpb.h
NVFLAGS := -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -cudart static \
  --expt-relaxed-constexpr -Xptxas -v

all: $(LIB)

$(LIB): $(SRCS) $(DEPS)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRCS) 2> build_ptxas.log || (cat build_ptxas.log; exit 1)
	@grep -E "registers|spill|bytes stack" build_ptxas.log | head -20

# Debug build with clock64 timelines of CTA 0 (scripts/trace_bwd.py); never shipped.
trace: dbg/libfcpb_trace.so
dbg/libfcpb_trace.so: $(SRCS) $(DEPS)
	@mkdir -p dbg
	$(NVCC) $(NVFLAGS) -DFCPB_TRACE -shared -o $@ $(SRCS) 2> dbg/ptxas.log || (cat dbg/ptxas.log; exit 1)

clean:
	rm -f $(LIB) build_ptxas.log dbg/libfcpb_trace.so

.PHONY: all clean trace

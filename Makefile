# Builds the in-tree CUDA library (sm_100a) and the oracle's reference-check helpers.
#   make -j8          -> paper_2309_04875_b200/lib/libhbrelu.so
NVCC    ?= nvcc
ARCH    ?= -gencode arch=compute_100a,code=sm_100a
NVFLAGS ?= -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O3 --expt-relaxed-constexpr $(ARCH)

CSRC    := paper_2309_04875_b200/csrc
OBJDIR  := build/obj
LIBDIR  := paper_2309_04875_b200/lib
LIB     := $(LIBDIR)/libhbrelu.so

WIDTH_TUS := $(wildcard $(CSRC)/hb_relu_w*.cu)
SRCS      := $(CSRC)/hb_api.cu $(CSRC)/hb_ops.cu $(CSRC)/hb_ring.cu $(CSRC)/hb_ring_tc.cu $(CSRC)/hb_conv_tma.cu $(CSRC)/hb_dealer.cu $(WIDTH_TUS)
OBJS      := $(patsubst $(CSRC)/%.cu,$(OBJDIR)/%.o,$(SRCS))
HDRS      := $(wildcard $(CSRC)/*.cuh) $(CSRC)/hb_widths.inc include/hb_relu.h

all: $(LIB)

$(OBJDIR)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(OBJS)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(ARCH) -shared -Xcompiler -fPIC $(OBJS) -o $@

clean:
	rm -rf build $(LIBDIR)

.PHONY: all clean

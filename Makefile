# Build the B200 (sm_100a) native library behind include/tb_bst.h.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 --expt-relaxed-constexpr
PKG := paper_1704_08364_b200
LIB := $(PKG)/lib/libtb_bst.so
SRC := $(PKG)/csrc/tb_api.cu
HDR := $(PKG)/csrc/tb_kernels.cuh $(PKG)/csrc/fft.cuh include/tb_bst.h

all: $(LIB)

$(LIB): $(SRC) $(HDR)
	@mkdir -p $(PKG)/lib
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC)

ptxas: $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c -o /tmp/tb_api.o $(SRC) 2>&1 | grep -E "Compiling|registers|spill" 

sass: $(LIB)
	cuobjdump -sass $(LIB) > profiles/sass_tb_bst.txt

clean:
	rm -f $(LIB)

.PHONY: all clean ptxas sass

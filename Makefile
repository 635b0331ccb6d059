# Build the B200 (sm_100a) native library behind include/tb_bst.h.
# tb_api.cu holds the plan / C ABI; tb_inst.cu is compiled once per radial
# length L (-DTB_L=<L>) so the kernel instantiations build in parallel.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 --expt-relaxed-constexpr
PKG := paper_1704_08364_b200
LIB := $(PKG)/lib/libtb_bst.so
OBJ := $(PKG)/build
CSRC := $(PKG)/csrc
HDR := $(CSRC)/tb_kernels.cuh $(CSRC)/fft.cuh $(CSRC)/tb_launch.cuh include/tb_bst.h
LS := 4 8 16 32 64 128 256 512 1024 2048 4096 8192 16384
INST := $(foreach l,$(LS),$(OBJ)/tb_inst_$(l).o)

all: $(LIB)

$(OBJ)/tb_api.o: $(CSRC)/tb_api.cu $(HDR)
	@mkdir -p $(OBJ)
	$(NVCC) $(NVFLAGS) -c -o $@ $<

$(OBJ)/tb_inst_%.o: $(CSRC)/tb_inst.cu $(HDR)
	@mkdir -p $(OBJ)
	$(NVCC) $(NVFLAGS) -DTB_L=$* -c -o $@ $<

$(LIB): $(OBJ)/tb_api.o $(INST)
	@mkdir -p $(PKG)/lib
	$(NVCC) $(ARCH) -shared -o $@ $^

# C99 client of the ABI (no Python): tests/c/abi_smoke.c
C_SMOKE := $(OBJ)/c_abi_smoke
c_smoke: $(C_SMOKE)
$(C_SMOKE): tests/c/abi_smoke.c include/tb_bst.h $(LIB)
	@mkdir -p $(OBJ)
	gcc -std=c99 -O2 -Wall -Wextra -D_DEFAULT_SOURCE -Iinclude -I/usr/local/cuda/include $< -o $@ \
	  -L$(PKG)/lib -ltb_bst -Wl,-rpath,'$$ORIGIN/../lib' -L/usr/local/cuda/lib64 -lcudart -lm

# registers / spills of the L = 4096 kernels
ptxas: $(CSRC)/tb_inst.cu $(HDR)
	$(NVCC) $(NVFLAGS) -DTB_L=4096 -Xptxas -v -c -o /tmp/tb_inst_4096.o $< 2>&1 | grep -E "Compiling|registers|spill"

sass: $(LIB)
	cuobjdump -sass $(OBJ)/tb_inst_4096.o > profiles/sass_tb_inst_4096.txt

clean:
	rm -rf $(LIB) $(OBJ)

.PHONY: all clean ptxas sass c_smoke

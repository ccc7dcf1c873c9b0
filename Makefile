# Build the B200 library (sm_100a) and the CPU oracle.
#   make            -> paper_1611_02445_b200/lib/libtlbm.so + oracle/build/liboracle.so
# -fmad=false keeps the reference's unfused multiply/add rounding (bit parity
# with the numpy reference); IEEE div/sqrt are nvcc defaults.
NVCC     ?= nvcc
PKG      := paper_1611_02445_b200
SRC      := $(wildcard $(PKG)/csrc/*.cu)
HDR      := $(wildcard $(PKG)/csrc/*.cuh) include/tlbm.h
LIB      := $(PKG)/lib/libtlbm.so
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  ?= -O3 -std=c++20 $(ARCH) -lineinfo -fmad=false -Xptxas -v \
            -Xcompiler -fPIC -Iinclude --expt-relaxed-constexpr

all: $(LIB) oracle

$(LIB): $(SRC) $(HDR)
	@mkdir -p $(PKG)/lib
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC) 2> $(PKG)/lib/ptxas.log || (cat $(PKG)/lib/ptxas.log; false)

oracle:
	$(MAKE) -s -C oracle

clean:
	rm -rf $(PKG)/lib oracle/build

.PHONY: all oracle clean

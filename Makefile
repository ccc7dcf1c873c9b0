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

all: oracle
	$(MAKE) -j8 $(LIB)

OBJ      := $(patsubst $(PKG)/csrc/%.cu,$(PKG)/lib/obj/%.o,$(SRC))

$(PKG)/lib/obj/%.o: $(PKG)/csrc/%.cu $(HDR)
	@mkdir -p $(PKG)/lib/obj
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> $@.log || (cat $@.log; false)

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ)
	@cat $(PKG)/lib/obj/*.o.log > $(PKG)/lib/ptxas.log

oracle:
	$(MAKE) -s -C oracle

clean:
	rm -rf $(PKG)/lib oracle/build

.PHONY: all oracle clean

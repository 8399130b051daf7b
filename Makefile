# Builds the C-ABI shared library of the hot path for sm_100a, and the
# oracle's C restatement (test infrastructure only).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
# bit-exact paths: no FMA contraction (the reference computes with plain
# IEEE adds/multiplies); the dense tile kernels opt back in per file.
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --fmad=false \
           --expt-extended-lambda -Iinclude
PKG := paper_1502_07451_b200
SRC := $(wildcard $(PKG)/csrc/*.cu)
OBJ := $(patsubst $(PKG)/csrc/%.cu,build/obj/%.o,$(SRC))
LIB := $(PKG)/libhetsched_b200.so

all: $(LIB)

build/obj/%.o: $(PKG)/csrc/%.cu $(wildcard $(PKG)/csrc/*.cuh) include/hetsched_b200.h
	@mkdir -p build/obj
	$(NVCC) $(NVFLAGS) $(if $(filter tile%,$*),--fmad=true,) -c $< -o $@

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -lcudart

clean:
	rm -rf build $(LIB)

.PHONY: all clean

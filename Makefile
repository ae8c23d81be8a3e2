# Builds the product library (sm_100a only) and the independent CPU oracle.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
# NCCL headers only (the library is dlopen-ed at run time by the band path)
NCCL_INC ?= $(firstword $(wildcard /opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/include) /usr/include)
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v -I$(NCCL_INC) --split-compile=0
PKG := paper_1505_00996_b200
LIB := $(PKG)/libfgf.so
SRCS := $(PKG)/csrc/fgf_api.cu
HDRS := $(wildcard $(PKG)/csrc/*.cuh) include/fgf.h
ORACLE := oracle/libfgf_oracle.so

all: $(LIB) $(ORACLE)

$(LIB): $(SRCS) $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRCS) -ldl 2> build/ptxas.log || (cat build/ptxas.log; false)

$(ORACLE): oracle/fgf_oracle.c
	gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fopenmp -shared -fPIC -o $@ $< -lm

clean:
	rm -f $(LIB) $(ORACLE)

.PHONY: all clean

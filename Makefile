# Builds the product library (sm_100a only) and the independent CPU oracle.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
# NCCL headers only (the library is dlopen-ed at run time by the band path)
NCCL_INC ?= $(firstword $(wildcard /opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/include) /usr/include)
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v -I$(NCCL_INC)
PKG := paper_1505_00996_b200
LIB := $(PKG)/libfgf.so
# one translation unit per kernel family, compiled in parallel (make -j), each in a single
# ptxas pass: nvcc --split-compile made register allocation depend on the split count
TUS := fgf_api fgf_k_mean fgf_k_out fgf_k_wide fgf_k_tiny fgf_k_apps fgf_k_lowres fgf_k_lowres_v3 fgf_k_lowres_v3h \
       fgf_k_lowres_v3bf fgf_k_lowres_v3b
OBJS := $(patsubst %,build/%.o,$(TUS))
HDRS := $(wildcard $(PKG)/csrc/*.cuh) include/fgf.h
ORACLE := oracle/libfgf_oracle.so
# test infrastructure: NCCL point-to-point stand-in for multi-process band tests on one GPU
SHIM := tests/libnccl_shim.so
CUDA_HOME ?= /usr/local/cuda

all: $(LIB) $(ORACLE) $(SHIM)

# K13 compiled through nvcc's split-compile path: there its loop and ring indices stay on the
# uniform datapath (550 uniform instructions vs 68), measured 4.14 -> 4.03 ms on config 4; the
# same path slows the strip engine's statistics kernel (0.564 -> 0.591 ms on config 3).
# nvcc hides the make jobserver's tokens from split-compile when it sees MAKEFLAGS (then it
# compiles unsplit, i.e. the other code), so the recipe runs it without MAKEFLAGS.
TUFLAGS_fgf_k_lowres := --split-compile=2
# the default fp32 variant alone in its unit: its split-compile code does not depend on the
# other instantiations (adding the 8-bit variants to the shared unit had changed it)

# the default K13 variant, one unit per sample type: the split-compile outcome with its
# indices on the uniform datapath (tools/nvcc_pick.py; nvcc's split-compile NVVM output varies
# from run to run)
K13_SYM = _ZN3fgf18lowres_gray_kernelILi1ELi4ELi9ELi17ELb0ELi160ELi3E$(1)EEvNS_12LowresParamsE
K13_fgf_k_lowres_v3 := $(call K13_SYM,f)
K13_fgf_k_lowres_v3h := $(call K13_SYM,6__half)
K13_fgf_k_lowres_v3bf := $(call K13_SYM,13__nv_bfloat16)
K13_fgf_k_lowres_v3b := $(call K13_SYM,h)
ELEM_fgf_k_lowres_v3 := float
ELEM_fgf_k_lowres_v3h := __half
ELEM_fgf_k_lowres_v3bf := __nv_bfloat16
ELEM_fgf_k_lowres_v3b := uint8_t
PICKED := fgf_k_lowres_v3 fgf_k_lowres_v3h fgf_k_lowres_v3bf fgf_k_lowres_v3b
# one source, fgf_k_lowres_v3.cu, compiled once per sample type
$(patsubst %,build/%.o,$(PICKED)): build/%.o: $(PKG)/csrc/fgf_k_lowres_v3.cu $(HDRS) Makefile tools/nvcc_pick.py
	@mkdir -p build
	python3 tools/nvcc_pick.py --out $@ --kernel $(K13_$*) -- $(NVCC) $(NVFLAGS) --split-compile=2 '-DFGF_V3_ELEM=$(ELEM_$*)' -c $< 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

build/%.o: $(PKG)/csrc/%.cu $(HDRS) Makefile
	@mkdir -p build
	env -u MAKEFLAGS -u MFLAGS $(NVCC) $(NVFLAGS) $(TUFLAGS_$*) -c -o $@ $< 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -ldl
	@cat $(patsubst %,build/%.ptxas.log,$(TUS)) > build/ptxas.log

$(ORACLE): oracle/fgf_oracle.c
	gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fopenmp -shared -fPIC -o $@ $< -lm

$(SHIM): tests/nccl_shim.cpp
	g++ -O2 -std=c++17 -shared -fPIC -I$(CUDA_HOME)/include -o $@ $< -L$(CUDA_HOME)/lib64 -lcudart

clean:
	rm -f $(LIB) $(ORACLE) $(SHIM)

.PHONY: all clean

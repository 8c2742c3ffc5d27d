# Builds the in-tree CUDA library (sm_100a only) and the CPU oracle.
#
#   make            -> paper_2410_18944_b200/libwostgpu.so + oracle/liboracle.so (+ oracle/_ref)
#
# -fmad=false: the walk path keeps the reference's fp64 operation order
# (no FMA contraction) so geometry and per-walk results are bit-comparable
# with the reference; kernels that do not need this use explicit fmaf().
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 \
           --expt-relaxed-constexpr -Xptxas -warn-spills $(EXTRA)
PKG := paper_2410_18944_b200
SRC := $(wildcard $(PKG)/csrc/*.cu)
HDR := $(wildcard $(PKG)/csrc/*.cuh $(PKG)/csrc/*.hpp) include/wostgpu.h include/wostgpu3.h include/wostgpu_types.h
OBJ := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRC))

all: $(PKG)/libwostgpu.so oracle

# translation units whose results are only statistically compared with the
# reference (tensor-core walk path, training) may contract FMAs
FAST_TUS := wg_walk_tc wg_walk_coop wg_train wg_train_tc wg3_walk_tc wg_wave2

build/%.o: $(PKG)/csrc/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) $(if $(filter $*,$(FAST_TUS)),-fmad=true,-fmad=false) -c $< -o $@

$(PKG)/libwostgpu.so: $(OBJ)
	$(NVCC) $(ARCH) -shared -Xlinker --no-undefined -o $@ $(OBJ) -lcudart -ldl

oracle:
	$(MAKE) -C oracle all

clean:
	rm -rf build $(PKG)/libwostgpu.so

.PHONY: all oracle clean

# diagnostic build: per-sub-phase clock64 totals of the tensor-core walk kernel
# (overwrites the library; rebuild with `make` afterwards)
# (the instrumented library is written over the normal one and its timestamp
# is backdated, so a later plain `make` relinks the normal library)
subprof: $(OBJ)
	$(NVCC) $(NVFLAGS) -fmad=true -DWG_SUBPROF -c $(PKG)/csrc/wg_walk_tc.cu -o build/wg_walk_tc_sub.o
	$(NVCC) $(ARCH) -shared -o $(PKG)/libwostgpu.so $(filter-out build/wg_walk_tc.o,$(OBJ)) build/wg_walk_tc_sub.o -lcudart -ldl
	touch -d '2000-01-01' $(PKG)/libwostgpu.so
.PHONY: subprof

# Build the in-tree C-ABI extension for sm_100a (B200).  `make` is what
# __graft_entry__.build() runs; the .so lands next to the Python package.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -Ipaper_2412_06198_b200/csrc \
           --expt-relaxed-constexpr -Xptxas -v $(EXTRA)
SRC := $(wildcard paper_2412_06198_b200/csrc/*.cu)
HDR := $(wildcard paper_2412_06198_b200/csrc/*.cuh paper_2412_06198_b200/csrc/*.h include/*.h)
OBJ := $(patsubst paper_2412_06198_b200/csrc/%.cu,build/%.o,$(SRC))
LIB := paper_2412_06198_b200/_sa_b200.so

all: $(LIB)

build/%.o: paper_2412_06198_b200/csrc/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.txt || (cat build/$*.ptxas.txt; false)

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -lcudart_static

# profiling variant: phase cycle counters in attn_fwd_kernel (tools/attn_prof.py)
PROF_LIB := paper_2412_06198_b200/_sa_b200_prof.so
PROF_OBJ := $(patsubst paper_2412_06198_b200/csrc/%.cu,build/prof/%.o,$(SRC))
build/prof/%.o: paper_2412_06198_b200/csrc/%.cu $(HDR)
	@mkdir -p build/prof
	$(NVCC) $(NVFLAGS) -DSA_ATTN_PROF -c $< -o $@ 2> build/prof/$*.ptxas.txt || (cat build/prof/$*.ptxas.txt; false)
$(PROF_LIB): $(PROF_OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(PROF_OBJ) -lcudart_static
prof: $(PROF_LIB)

clean:
	rm -rf build $(LIB)

.PHONY: all clean prof

# A/B variant: attention epilogue through a TMA-store stage (SA_ATTN_TMA_STORE=1)
TMA_LIB := paper_2412_06198_b200/_sa_b200_tma.so
build/tma/attn_fwd.o: paper_2412_06198_b200/csrc/attn_fwd.cu $(HDR)
	@mkdir -p build/tma
	$(NVCC) $(NVFLAGS) -DSA_ATTN_TMA_STORE=1 -c $< -o $@ 2> build/tma/attn_fwd.ptxas.txt || (cat build/tma/attn_fwd.ptxas.txt; false)
$(TMA_LIB): build/tma/attn_fwd.o $(filter-out build/attn_fwd.o,$(OBJ))
	$(NVCC) $(ARCH) -shared -o $@ $^ -lcudart_static
tma: $(TMA_LIB)
.PHONY: tma

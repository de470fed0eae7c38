# Builds the in-tree C-ABI library paper_2507_01004_b200/libzeco_gla.so (sm_100a)
# and the oracle's compiled helpers.  `python -c "import __graft_entry__ as g; g.build()"`
# runs the same recipe.
NVCC ?= nvcc
PKG := paper_2507_01004_b200
SRC := $(wildcard $(PKG)/csrc/*.cu)
HDR := $(wildcard $(PKG)/csrc/*.cuh $(PKG)/csrc/*.h) include/zeco_gla.h
NVFLAGS := -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
           -Xcompiler -fPIC --expt-relaxed-constexpr \
           -Xptxas -v -DZGLA_BUILD
OBJ := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRC))

all: $(PKG)/libzeco_gla.so

build/%.o: $(PKG)/csrc/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(PKG)/libzeco_gla.so: $(OBJ)
	$(NVCC) -gencode arch=compute_100a,code=sm_100a -shared -o $@ $(OBJ) -lcuda

clean:
	rm -rf build $(PKG)/libzeco_gla.so

.PHONY: all clean

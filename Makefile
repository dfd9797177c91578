# libpoba: sm_100a only.  `make` builds paper_2204_12834_b200/lib/libpoba.so in-tree.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall --expt-relaxed-constexpr
SRC := $(wildcard paper_2204_12834_b200/csrc/*.cu)
CPPSRC := $(wildcard paper_2204_12834_b200/csrc/*.cpp)
OBJ := $(patsubst paper_2204_12834_b200/csrc/%.cu,build/%.o,$(SRC)) $(patsubst paper_2204_12834_b200/csrc/%.cpp,build/%.o,$(CPPSRC))
CXX ?= g++
CXXFLAGS := -O3 -std=c++17 -fPIC -Wall
LIB := paper_2204_12834_b200/lib/libpoba.so

ORACLE_LIB := oracle/lib/libpoba_oracle.so
all: $(LIB) oracle

build/%.o: paper_2204_12834_b200/csrc/%.cu paper_2204_12834_b200/csrc/poba_internal.h include/poba.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

build/%.o: paper_2204_12834_b200/csrc/%.cpp include/poba.h
	@mkdir -p build
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(LIB): $(OBJ)
	@mkdir -p paper_2204_12834_b200/lib
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -lcudart -ldl

# test infrastructure: the C restatement of the W / W^T passes (oracle/poba_term.c)
oracle: $(ORACLE_LIB)

$(ORACLE_LIB): oracle/poba_term.c
	@mkdir -p oracle/lib
	gcc -O2 -fPIC -shared -fopenmp -o $@ $<

ptxas:
	@for f in $(SRC); do $(NVCC) $(NVFLAGS) -Xptxas -v -c $$f -o /dev/null 2>&1 | grep -E "Function properties|registers|spill|Compiling entry" ; done

clean:
	rm -rf build $(LIB) $(ORACLE_LIB)

.PHONY: all clean ptxas oracle

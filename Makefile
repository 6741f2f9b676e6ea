# Builds the sm_100a CUDA library behind the C ABI (include/hankelfft_b200.h)
# and the oracle's checker pieces.  `python -c "import __graft_entry__ as g; g.build()"`
# runs this.  Objects go to build/, the shared library next to the package.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -std=c++17 -O3 --expt-relaxed-constexpr $(ARCH) -lineinfo -Xcompiler -fPIC \
           -Xptxas -warn-spills
SRC := paper_1401_6238_b200/csrc
OBJ := build/obj
LIB := paper_1401_6238_b200/libhankelfft_b200.so

CU := $(wildcard $(SRC)/*.cu)
OBJS := $(patsubst $(SRC)/%.cu,$(OBJ)/%.o,$(CU))
HDRS := $(wildcard $(SRC)/*.cuh) $(wildcard $(SRC)/*.h) include/hankelfft_b200.h

all: $(LIB)

# per-file ptxas options: the ping-pong kernel keeps 3 transforms' worth of
# swizzled addresses live under -O3 scheduling and spills at 128 registers;
# ptxas -O1 schedules it in 125 registers with no spills.
PTXAS_hk_pp1d := -Xptxas -O1

$(OBJ)/%.o: $(SRC)/%.cu $(HDRS) Makefile
	@mkdir -p $(OBJ)
	$(NVCC) $(NVFLAGS) $(PTXAS_$*) -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart_static -lrt -lpthread -ldl

clean:
	rm -rf build $(LIB)

.PHONY: all clean

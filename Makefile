# Build the B200 (sm_100a) shared library behind the C ABI in include/fc2.h.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr $(EXTRA)
PKG := paper_2508_03760_b200
SRC := $(PKG)/csrc
OBJ := $(PKG)/_build

LIB := $(PKG)/libfc2.so
OBJS := $(OBJ)/fc2_codec.o $(OBJ)/fc2_comm.o $(OBJ)/fc2_moe.o $(patsubst $(SRC)/%.cu,$(OBJ)/%.o,$(wildcard $(SRC)/fc2_inst_b*.cu))

all: $(LIB)

$(OBJ)/%.o: $(SRC)/%.cu $(wildcard $(SRC)/*.cuh) include/fc2.h
	@mkdir -p $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@ > $(OBJ)/$*.ptxas.log 2>&1 || (cat $(OBJ)/$*.ptxas.log; false)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS)

clean:
	rm -rf $(OBJ) $(LIB)

.PHONY: all clean

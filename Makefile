# Builds the in-tree CUDA library for sm_100a (B200) and the oracle's C helpers.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v $(EXTRA)
SRC := paper_1112_3010_b200/csrc
OBJ := build/obj
LIB := paper_1112_3010_b200/_lib/libeikfld_b200.so
UNITS := pipeline launch_col_sparse launch_col_dense launch_col_spec launch_lines launch_rows classify dd_pipeline spectral
OBJS := $(addprefix $(OBJ)/,$(addsuffix .o,$(UNITS))) $(OBJ)/dd_twiddle.o
HDRS := $(wildcard $(SRC)/*.cuh) include/eikfld_b200.h

all: $(LIB)

$(OBJ)/%.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@ > $@.ptxas.log 2>&1 || (cat $@.ptxas.log; exit 1)

# host-only helper (binary128 twiddles for the double-double path)
$(OBJ)/dd_twiddle.o: $(SRC)/dd_twiddle.cpp
	@mkdir -p $(OBJ)
	g++ -O2 -fPIC -c $< -o $@

$(LIB): $(OBJS)
	@mkdir -p $(dir $(LIB))
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -Xlinker -Bstatic -lquadmath -Xlinker -Bdynamic

clean:
	rm -rf build $(LIB)

.PHONY: all clean

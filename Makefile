# Build of the B200-native CPAA library (sm_100a only) and the CPU checkers.
#   make            -> paper_2112_01743_b200/lib/libchebpr_b200.so + oracle
NVCC      ?= nvcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC,-ffp-contract=off \
             --expt-extended-lambda -Iinclude -Xptxas -warn-spills
SRC_DIR   := paper_2112_01743_b200/csrc
LIB_DIR   := paper_2112_01743_b200/lib
OBJ_DIR   := build/obj
SRCS      := $(SRC_DIR)/build.cu $(SRC_DIR)/cpaa.cu $(SRC_DIR)/capi.cu $(SRC_DIR)/generate.cu $(SRC_DIR)/spmm.cu $(SRC_DIR)/coeffs.cpp
OBJS      := $(patsubst $(SRC_DIR)/%,$(OBJ_DIR)/%.o,$(SRCS))
HDRS      := $(SRC_DIR)/common.cuh $(SRC_DIR)/device.cuh include/chebpr_cuda.h

all: $(LIB_DIR)/libchebpr_b200.so oracle

$(OBJ_DIR)/%.cu.o: $(SRC_DIR)/%.cu $(HDRS)
	@mkdir -p $(OBJ_DIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(OBJ_DIR)/%.cpp.o: $(SRC_DIR)/%.cpp $(HDRS)
	@mkdir -p $(OBJ_DIR)
	$(NVCC) $(NVFLAGS) -x cu -c $< -o $@

$(LIB_DIR)/libchebpr_b200.so: $(OBJS)
	@mkdir -p $(LIB_DIR)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart -lnccl

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(LIB_DIR)
	$(MAKE) -C oracle clean

.PHONY: all oracle clean

# Build of the B200-native CPAA library (sm_100a only) and the CPU checkers.
#   make            -> paper_2112_01743_b200/lib/libchebpr_b200.so + oracle
NVCC      ?= nvcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
EXP       ?= 0
NVFLAGS   := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC,-ffp-contract=off \
             --expt-extended-lambda -Iinclude -Xptxas -warn-spills -DCHEB_TERM_EXPERIMENTS=$(EXP)
SRC_DIR   := paper_2112_01743_b200/csrc
LIB_DIR   := paper_2112_01743_b200/lib
OBJ_DIR   := build/obj
SRCS      := $(SRC_DIR)/build.cu $(SRC_DIR)/cpaa.cu $(SRC_DIR)/dist.cu $(SRC_DIR)/power.cu $(SRC_DIR)/capi.cu $(SRC_DIR)/generate.cu $(SRC_DIR)/spmm.cu $(SRC_DIR)/ingest.cu $(SRC_DIR)/validate.cu $(SRC_DIR)/coeffs.cpp
OBJS      := $(patsubst $(SRC_DIR)/%,$(OBJ_DIR)/%.o,$(SRCS))
REFTEST_SRC ?= /root/reference/proj/tests
REFTESTS    := test_coefficients test_graph test_cpaa test_power test_metrics
HDRS      := $(SRC_DIR)/common.cuh $(SRC_DIR)/device.cuh $(SRC_DIR)/term.cuh include/chebpr_cuda.h
# NCCL: the copy torch ships (nvidia-nccl wheel), so that this library and torch resolve
# libnccl.so.2 to the same build whichever is loaded first; the system one otherwise.
NCCL_LIB  := $(shell python -c "import nvidia.nccl, os; print(os.path.join(list(nvidia.nccl.__path__)[0], 'lib'))" 2>/dev/null)
LDNCCL    := $(if $(NCCL_LIB),-L$(NCCL_LIB) -l:libnccl.so.2 -Xlinker -rpath -Xlinker $(NCCL_LIB),-lnccl)

BIN_DIR   := paper_2112_01743_b200/bin
CLI       := $(abspath $(BIN_DIR))/chebpr

all: $(LIB_DIR)/libchebpr_b200.so $(LIB_DIR)/libchebpr_dropin.so $(BIN_DIR)/chebpr oracle $(if $(wildcard $(REFTEST_SRC)/test_cpaa.cpp),reftests,)

$(OBJ_DIR)/%.cu.o: $(SRC_DIR)/%.cu $(HDRS)
	@mkdir -p $(OBJ_DIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(OBJ_DIR)/%.cpp.o: $(SRC_DIR)/%.cpp $(HDRS)
	@mkdir -p $(OBJ_DIR)
	$(NVCC) $(NVFLAGS) -x cu -c $< -o $@

$(LIB_DIR)/libchebpr_b200.so: $(OBJS)
	@mkdir -p $(LIB_DIR)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart $(LDNCCL)

# C++ drop-in layer (the reference's chebpr:: API over the C-ABI)
$(LIB_DIR)/libchebpr_dropin.so: $(SRC_DIR)/dropin.cpp $(SRC_DIR)/csv.cpp $(wildcard include/chebpr/*.hpp) include/chebpr_cuda.h $(LIB_DIR)/libchebpr_b200.so
	g++ -std=c++20 -O2 -fPIC -shared -ffp-contract=off -Wall -Wextra -pthread -Iinclude -o $@ $(SRC_DIR)/dropin.cpp \
	    $(SRC_DIR)/csv.cpp -L$(LIB_DIR) -lchebpr_b200 -Wl,-rpath,'$$ORIGIN'

# `chebpr` CLI (gen / run / compare / coeffs) over the C-ABI + drop-in
$(BIN_DIR)/chebpr: $(SRC_DIR)/cli.cpp $(LIB_DIR)/libchebpr_dropin.so
	@mkdir -p $(BIN_DIR)
	g++ -std=c++20 -O2 -Wall -Wextra -Iinclude -o $@ $(SRC_DIR)/cli.cpp \
	    -L$(LIB_DIR) -lchebpr_dropin -lchebpr_b200 -Wl,-rpath,'$$ORIGIN/../lib'

# The reference's own doctest suites compiled UNCHANGED against the drop-in (test
# infrastructure; sources read in place from /root/reference, binaries into build/reftests).
reftests: $(addprefix build/reftests/,$(REFTESTS)) build/reftests/acceptance_main build/reftests/test_cli

# The reference's acceptance gate (9 criteria) and CLI suite, unchanged, driving our `chebpr`
# binary (CHEBPR_CLI_PATH, as the reference's CMake sets it to its own CLI).
build/reftests/acceptance_main: $(REFTEST_SRC)/acceptance_main.cpp $(LIB_DIR)/libchebpr_dropin.so $(BIN_DIR)/chebpr tests/cpp/doctest.h
	@mkdir -p build/reftests
	g++ -std=c++20 -O2 -Iinclude -Itests/cpp -I$(REFTEST_SRC) '-DCHEBPR_CLI_PATH="$(CLI)"' -o $@ $< \
	    -L$(LIB_DIR) -lchebpr_dropin -lchebpr_b200 -Wl,-rpath,'$$ORIGIN/../../$(LIB_DIR)' 

build/reftests/test_cli: $(REFTEST_SRC)/test_cli.cpp $(LIB_DIR)/libchebpr_dropin.so $(BIN_DIR)/chebpr tests/cpp/doctest.h
	@mkdir -p build/reftests
	g++ -std=c++20 -O2 -Iinclude -Itests/cpp -I$(REFTEST_SRC) '-DCHEBPR_CLI_PATH="$(CLI)"' -o $@ $< \
	    -L$(LIB_DIR) -lchebpr_dropin -lchebpr_b200 -Wl,-rpath,'$$ORIGIN/../../$(LIB_DIR)'

build/reftests/%: $(REFTEST_SRC)/%.cpp $(LIB_DIR)/libchebpr_dropin.so tests/cpp/doctest.h
	@mkdir -p build/reftests
	g++ -std=c++20 -O2 -Iinclude -Itests/cpp -I$(REFTEST_SRC) -o $@ $< \
	    -L$(LIB_DIR) -lchebpr_dropin -lchebpr_b200 -Wl,-rpath,'$$ORIGIN/../../$(LIB_DIR)'

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(LIB_DIR) $(BIN_DIR)
	$(MAKE) -C oracle clean

print-ldnccl:
	@echo $(LDNCCL)

.PHONY: all oracle clean reftests print-ldnccl

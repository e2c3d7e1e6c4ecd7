# B200-native Crystal: builds the product library and the (test-only) checkers.
#   make            -> paper_2003_01178_b200/libcrystal_b200.so + oracle/
#   make lib        -> product library only
NVCC      ?= /usr/local/cuda/bin/nvcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-Wall -Iinclude $(EXTRA) \
             -Xptxas -v --expt-relaxed-constexpr
CSRC      := paper_2003_01178_b200/csrc
BUILD     := build/obj
LIB       := paper_2003_01178_b200/libcrystal_b200.so
CU_SRCS   := $(wildcard $(CSRC)/*.cu)
CPP_SRCS  := $(wildcard $(CSRC)/*.cpp)
OBJS      := $(patsubst $(CSRC)/%.cu,$(BUILD)/%.o,$(CU_SRCS)) \
             $(patsubst $(CSRC)/%.cpp,$(BUILD)/%.o,$(CPP_SRCS))
HDRS      := $(wildcard $(CSRC)/*.cuh) $(wildcard $(CSRC)/*.hpp) include/crystal_b200.h

all: lib oracle

lib: $(LIB)

$(BUILD)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(BUILD)/$*.ptxas.txt || (cat $(BUILD)/$*.ptxas.txt; false)

$(BUILD)/%.o: $(CSRC)/%.cpp $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -x cu -c $< -o $@ 2> $(BUILD)/$*.ptxas.txt || (cat $(BUILD)/$*.ptxas.txt; false)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(OBJS) -ldl

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(LIB)
	$(MAKE) -C oracle clean

.PHONY: all lib oracle clean

# hetsim-b200 build.
#
#   make            -> paper_2009_07482_b200/libhetsim.so   (product: C++ host runtime +
#                                                            hs_* C ABI + sm_100a kernels)
#   make oracle     -> oracle/liboracle.so, oracle/_ref/libhetsim_ref.so (test checkers)
#
# nvcc cross-compiles for sm_100a without a GPU. `-arch=sm_100a` is not used on
# purpose: tcgen05 PTX needs the arch-specific target on both stages.
NVCC     ?= /usr/local/cuda/bin/nvcc
CXX      ?= g++
PKG      := paper_2009_07482_b200
SRC      := $(PKG)/csrc
BUILD    := build
ARCH     := -gencode arch=compute_100a,code=sm_100a
CXXFLAGS := -std=c++20 -O2 -fPIC -Wall -Wextra -Iinclude -I$(SRC)
NVEXTRA  ?=
NVFLAGS  := -std=c++20 -O3 $(ARCH) -lineinfo -Xcompiler -fPIC -Iinclude -I$(SRC) -Xptxas -v $(NVEXTRA)

CPP_SRCS := $(wildcard $(SRC)/core/*.cpp) $(wildcard $(SRC)/sched/*.cpp) \
            $(wildcard $(SRC)/capi/*.cpp) $(wildcard $(SRC)/exec/*.cpp)
CU_SRCS  := $(wildcard $(SRC)/cuda/*.cu)
CPP_OBJS := $(patsubst $(SRC)/%.cpp,$(BUILD)/%.o,$(CPP_SRCS))
CU_OBJS  := $(patsubst $(SRC)/%.cu,$(BUILD)/%.o,$(CU_SRCS))
HEADERS  := $(wildcard include/*.h) $(wildcard include/hetsim/*.hpp) $(wildcard $(SRC)/*/*.hpp) \
            $(wildcard $(SRC)/*/*.cuh)

LIB := $(PKG)/libhetsim.so

all: $(LIB)

$(BUILD)/%.o: $(SRC)/%.cpp $(HEADERS)
	@mkdir -p $(dir $@)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(BUILD)/%.o: $(SRC)/%.cu $(HEADERS)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(BUILD)/$(notdir $<).ptxas.txt || (cat $(BUILD)/$(notdir $<).ptxas.txt; false)

$(LIB): $(CPP_OBJS) $(CU_OBJS)
	$(NVCC) $(ARCH) -shared -Xcompiler -fPIC -Xlinker -Bsymbolic -o $@ $^ -lpthread

oracle:
	$(MAKE) -C oracle oracle
	@if [ -d /root/reference/proj/src ]; then $(MAKE) -C oracle ref; else echo "reference sources absent: using prebuilt oracle/_ref"; fi

clean:
	rm -rf $(BUILD) $(LIB)

.PHONY: all oracle clean

# Host race check: the C++ runtime (spec model, scheduler, engine,
# callback -> MPSC queue -> Scheduler::cb) built with ThreadSanitizer, linked with
# the sm_100a kernels and the drop-in driver tests/cxx/dropin_main.cpp (Alg. 1 in
# dynamic mode through hetsim::CudaExecutor: CUDA host callbacks deliver completions).
TSAN_BUILD := build_tsan
TSAN_CXX   ?= $(shell command -v g++-13 || echo $(CXX))
TSAN_OBJS  := $(patsubst $(SRC)/%.cpp,$(TSAN_BUILD)/%.o,$(CPP_SRCS))
TSAN_EXE   := $(TSAN_BUILD)/dropin_tsan

$(TSAN_BUILD)/%.o: $(SRC)/%.cpp $(HEADERS)
	@mkdir -p $(dir $@)
	$(TSAN_CXX) $(CXXFLAGS) -g -O1 -fsanitize=thread -c $< -o $@

$(TSAN_EXE): tests/cxx/dropin_main.cpp $(TSAN_OBJS) $(CU_OBJS)
	$(TSAN_CXX) -std=c++20 -g -O1 -fsanitize=thread -Iinclude $< $(TSAN_OBJS) $(CU_OBJS) \
	    -L/usr/local/cuda/lib64 -lcudart_static -ldl -lrt -lpthread -o $@

tsan: $(TSAN_EXE)

.PHONY: tsan

# Build recipe for the B200 library, the CPU oracle and the reference build.
#   make            liblrb.so (sm_100a) + oracle/liblrb_oracle.so (+ oracle/_ref when the reference is present)
#   make lib        only the CUDA library
#   make oracle     only the C oracle
#   make ref        only oracle/_ref (needs /root/reference)
NVCC      ?= nvcc
CC        ?= gcc
CXX       ?= g++
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
             -Xptxas -warn-spills --expt-relaxed-constexpr
PKG       := paper_2311_07602_b200
CSRC      := $(PKG)/csrc
BUILD     := build/obj
LIB       := $(PKG)/liblrb.so
CU_SRCS   := $(wildcard $(CSRC)/*.cu)
CU_OBJS   := $(patsubst $(CSRC)/%.cu,$(BUILD)/%.o,$(CU_SRCS))
HDRS      := $(wildcard $(CSRC)/*.cuh) $(wildcard $(CSRC)/*.h) include/lrb.h include/lrb_rng.h

REFERENCE ?= /root/reference
REF_INC   := $(REFERENCE)/proj/include
# The reference builds with -O3 -march=native (proj/CMakeLists.txt:13-20). The
# built .so travels to the GPU box, whose host CPU may differ, so the portable
# x86-64-v3 level (AVX2 + FMA) stands in for native: the oracle loop is a
# scalar FMA chain either way.
REF_FLAGS := -std=c++20 -O3 -march=x86-64-v3 -fPIC -shared -pthread

.PHONY: all lib oracle ref clean
all: lib oracle $(if $(wildcard $(REF_INC)/lrbatch/dense.hpp),ref,)

lib: $(LIB)
oracle: oracle/liblrb_oracle.so
ref: oracle/_ref/liblrb_ref.so

$(BUILD)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@

# exported symbols are exactly the extern "C" lrb_* entry points
$(LIB): $(CU_OBJS) $(CSRC)/lrb.map
	$(NVCC) $(ARCH) -shared -Xcompiler -fPIC $(CU_OBJS) -o $@ -Xlinker --exclude-libs=ALL -Xlinker --version-script=$(CSRC)/lrb.map

oracle/liblrb_oracle.so: oracle/lrb_oracle.c oracle/lrb_oracle.h include/lrb_rng.h
	$(CC) -std=c11 -O2 -fPIC -shared -pthread -ffp-contract=off -Iinclude $< -o $@ -lm

oracle/_ref/liblrb_ref.so: oracle/ref_shim.cpp
	@mkdir -p oracle/_ref
	$(CXX) $(REF_FLAGS) -I$(REF_INC) -Iinclude -DLRBATCH_MACHINE_DIR=\"$(REFERENCE)/proj/machines\" $< -o $@

clean:
	rm -rf $(BUILD) $(LIB) oracle/liblrb_oracle.so oracle/_ref

# Builds the product library (CUDA, sm_100a) and the oracle (plain C, test infrastructure).
NVCC     ?= nvcc
PKG      := paper_2301_06284_b200
NCCL_DIR ?= /opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall -Iinclude -I$(NCCL_DIR)/include \
            --expt-relaxed-constexpr -Xptxas -warn-spills $(EXTRA)
SRCS     := $(wildcard $(PKG)/csrc/*.cu)
OBJS     := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRCS))
HDRS     := $(wildcard $(PKG)/csrc/*.cuh) include/rgnn.h

all: $(PKG)/librgnn.so oracle/liboracle.so

build/%.o: $(PKG)/csrc/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(PKG)/librgnn.so: $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -L$(NCCL_DIR)/lib -l:libnccl.so.2 -Xlinker -rpath=$(NCCL_DIR)/lib -lcudart

oracle/liboracle.so: oracle/rgnn_oracle.c
	gcc -O2 -fopenmp -fPIC -shared -std=c11 -Wall -o $@ $< -lm

clean:
	rm -rf build $(PKG)/librgnn.so oracle/liboracle.so

.PHONY: all clean

# In-tree build of the three native libraries.
#   paper_cs_0609090_b200/libldpc.so  -- the product: CUDA kernels for sm_100a + C ABI (include/ldpc.h)
#   oracle/liboracle.so                -- CPU oracle (test infrastructure only)
#   ldpcgen/libldpcgen.so              -- seeded input generators
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
LIB := paper_cs_0609090_b200/libldpc.so
CSRC := paper_cs_0609090_b200/csrc
SRCS := $(wildcard $(CSRC)/*.cu)
OBJS := $(patsubst $(CSRC)/%.cu,build/%.o,$(SRCS))
HDRS := $(wildcard $(CSRC)/*.cuh) $(wildcard $(CSRC)/*.h) include/ldpc.h

all: $(LIB) oracle/liboracle.so ldpcgen/libldpcgen.so examples/decode_c

build/%.o: $(CSRC)/%.cu $(HDRS)
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart

oracle/liboracle.so: oracle/oracle.c oracle/engine.inc
	gcc -O2 -std=gnu11 -fPIC -shared -ffp-contract=off -o $@ oracle/oracle.c -lm -lpthread

ldpcgen/libldpcgen.so: ldpcgen/ldpcgen.c
	gcc -O2 -std=gnu11 -fPIC -shared -ffp-contract=off -o $@ ldpcgen/ldpcgen.c -lm -lpthread

# plain-C consumer of the C ABI (examples/decode_c.c)
CUDA_HOME ?= /usr/local/cuda
examples/decode_c: examples/decode_c.c include/ldpc.h $(LIB)
	gcc -O2 -std=c11 -Wall -Iinclude -I$(CUDA_HOME)/include -o $@ $< -Lpaper_cs_0609090_b200 -lldpc \
	  -L$(CUDA_HOME)/lib64 -lcudart -Wl,-rpath,'$$ORIGIN/../paper_cs_0609090_b200' -Wl,-rpath,$(CUDA_HOME)/lib64

# checked build: device-side bounds checks (LDPC_CHECK in csrc/args.cuh) on the hot loops.
# LDPC_LIBRARY=$(CURDIR)/build/checked/libldpc.so python -m pytest tests -m gpu
CHK_OBJS := $(patsubst $(CSRC)/%.cu,build/checked/%.o,$(SRCS))
build/checked/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p build/checked
	$(NVCC) $(NVFLAGS) -DLDPC_CHECKED -c -o $@ $< 2> build/checked/$*.ptxas.log || (cat build/checked/$*.ptxas.log; false)
build/checked/libldpc.so: $(CHK_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(CHK_OBJS) -lcudart
checked: build/checked/libldpc.so

clean:
	rm -f build/*.o $(LIB) oracle/liboracle.so ldpcgen/libldpcgen.so examples/decode_c

.PHONY: all clean checked
$(shell mkdir -p build)

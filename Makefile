# Build libspa.so (the C-ABI product, include/spa.h) without Python:  make            -> paper_2511_12056_b200/lib/libspa.so
#                                                                    make c-abi-test -> builds and runs tests/c_abi/abi_smoke.c
# Same flags as paper_2511_12056_b200/_build.py (which __graft_entry__.build() uses).
NVCC    ?= /usr/local/cuda/bin/nvcc
PYTHON  ?= python
NCCL    ?= $(shell $(PYTHON) -c "import nvidia.nccl as n; print(list(n.__path__)[0])")
ARCH    := -gencode arch=compute_100a,code=sm_100a
CSRC    := paper_2511_12056_b200/csrc
LIBDIR  := paper_2511_12056_b200/lib
OBJS    := $(LIBDIR)/attn_fwd.o $(LIBDIR)/qkv_gemm.o $(LIBDIR)/reshard.o $(LIBDIR)/lse_merge.o $(LIBDIR)/nccl_window.o \
           $(LIBDIR)/spa_api.o
CUFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -I$(NCCL)/include -Iinclude

all: $(LIBDIR)/libspa.so

$(LIBDIR)/%.o: $(CSRC)/%.cu $(CSRC)/ptx.cuh $(CSRC)/spa_internal.h include/spa.h
	@mkdir -p $(LIBDIR)
	$(NVCC) $(CUFLAGS) -x cu -c $< -o $@

$(LIBDIR)/spa_api.o: $(CSRC)/spa_api.cpp $(CSRC)/spa_internal.h include/spa.h
	@mkdir -p $(LIBDIR)
	$(NVCC) $(ARCH) -O3 -std=c++17 -Xcompiler -fPIC,-O3 -I$(NCCL)/include -Iinclude -c $< -o $@

$(LIBDIR)/libspa.so: $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -L$(NCCL)/lib -l:libnccl.so.2 -Xlinker=-rpath=$(NCCL)/lib \
	    -lcudart_static -ldl -lrt -lpthread

c-abi-test: $(LIBDIR)/libspa.so
	gcc -std=c11 -O1 -Iinclude tests/c_abi/abi_smoke.c $(LIBDIR)/libspa.so -o /tmp/spa_abi_smoke \
	    -Wl,-rpath,$(abspath $(LIBDIR))
	/tmp/spa_abi_smoke

clean:
	rm -f $(OBJS) $(LIBDIR)/libspa.so

.PHONY: all c-abi-test clean

# Build of libswb200.so (sm_100a only).  The oracle (oracle/decoder.py) is
# fp32 torch on the CPU and needs no build.
#   make            -> paper_2311_18677_b200/libswb200.so
#   make sass       -> dump SASS of the library (proof of UTCHMMA / UTMALDG)
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr \
           -Xptxas -v
SRC := paper_2311_18677_b200/csrc
OBJDIR := build/obj
CU := $(wildcard $(SRC)/*.cu)
CPP := $(wildcard $(SRC)/*.cpp)
OBJ := $(patsubst $(SRC)/%.cu,$(OBJDIR)/%.o,$(CU)) $(patsubst $(SRC)/%.cpp,$(OBJDIR)/%.o,$(CPP))
LIB := paper_2311_18677_b200/libswb200.so

all: $(LIB)

$(OBJDIR)/%.o: $(SRC)/%.cu $(SRC)/common.cuh include/swb200.h
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(OBJDIR)/$*.ptxas.txt || (cat $(OBJDIR)/$*.ptxas.txt; false)

$(OBJDIR)/%.o: $(SRC)/%.cpp include/swb200.h
	@mkdir -p $(OBJDIR)
	$(NVCC) -O3 -std=c++17 -Xcompiler -fPIC -c $< -o $@

$(LIB): $(OBJ)
	$(NVCC) -shared $(ARCH) -o $@ $(OBJ) -cudart static

sass: $(LIB)
	/usr/local/cuda/bin/cuobjdump -sass $(LIB) > build/libswb200.sass
	@grep -c UTCHMMA build/libswb200.sass || true
	@grep -c UTMALDG build/libswb200.sass || true

clean:
	rm -rf build $(LIB)

.PHONY: all clean sass

# timeline-probe build of the decode attention (tools/attn_probe.py only):
# build/var/libswb200_probe.so, copied over the library on a GPU box for a run
probe-lib: $(OBJ)
	@mkdir -p build/var
	$(NVCC) $(NVFLAGS) -DSWB_ATTN_PROBE -c $(SRC)/attention.cu -o build/var/attention_probe.o
	$(NVCC) -shared $(ARCH) -o build/var/libswb200_probe.so $(filter-out $(OBJDIR)/attention.o,$(OBJ)) build/var/attention_probe.o -cudart static

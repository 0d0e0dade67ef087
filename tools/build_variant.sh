#!/bin/bash
# Build a variant of libarctopk.so with extra nvcc -D flags into ab/<name>/ (A/B timing):
#   bash tools/build_variant.sh ld1 -DARC_SK_LD=1
set -e
name=$1; shift
mkdir -p ab/$name
NCCL_INC=$(python -c "import nvidia.nccl,os;print(os.path.join(nvidia.nccl.__path__[0],'include'))")
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -ftz=false -prec-div=true \
  -prec-sqrt=true -Xcompiler -fPIC -shared -cudart static -Iinclude -I$NCCL_INC "$@" \
  paper_2510_26709_b200/csrc/arc_kernels.cu paper_2510_26709_b200/csrc/arc_sketch.cu paper_2510_26709_b200/csrc/arc_select.cu \
  paper_2510_26709_b200/csrc/arc_lsa.cu paper_2510_26709_b200/csrc/arc_optim.cu paper_2510_26709_b200/csrc/arc_loopback.cu \
  paper_2510_26709_b200/csrc/arc_api.cu -o ab/$name/libarctopk.so -ldl
echo ab/$name/libarctopk.so

#!/bin/bash
# Build a variant of libarctopk.so with extra nvcc -D flags into ab/<name>/ (A/B timing):
#   bash tools/build_variant.sh ld1 -DARC_SK_LD=1
set -e
name=$1; shift
mkdir -p ab/$name
python -m paper_2510_26709_b200._build --out ab/$name/libarctopk.so "$@"

#!/bin/bash
# Build a profiling variant of the product library with extra nvcc flags into _exp/<name>.so
# (git-ignored; travels to the GPU box) for in-process A/B timing with tools/tune_fwd.py:
#   tools/build_variant.sh ablate -DDASMC_EPI_ABLATIONS
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
mkdir -p "$root/_exp"
make -C "$root/paper_2601_21983_b200" -s -j4 BUILD="$root/_exp/build_$name" LIB="$root/_exp/$name.so" EXTRA="$*"

#!/bin/bash
# build_variant.sh <tag> [extra nvcc flags...] -> paper_2205_11226_b200/_blockmend_b200.<tag>.so
set -e
cd "$(dirname "$0")/.."
tag=$1; shift
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared "$@" \
  -o paper_2205_11226_b200/_blockmend_b200.$tag.so paper_2205_11226_b200/csrc/bm_conceal.cu paper_2205_11226_b200/csrc/bm_conceal_wide.cu paper_2205_11226_b200/csrc/bm_conceal_cluster.cu paper_2205_11226_b200/csrc/bm_aux.cu paper_2205_11226_b200/csrc/bm_api.cu

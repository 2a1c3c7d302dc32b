#!/bin/bash
# ptxas register/spill report for one kernel-name pattern in ops.cu (sm_100a): scripts/ptxas_check.sh <regex>
cd "$(dirname "$0")/../paper_2303_10233_b200/csrc" && nvcc -c -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xptxas -v ${2:-ops.cu} -o /tmp/ptxas_check.o 2>&1 | grep -E "error|$1" -A2 | grep -E "error|registers|spill|Compiling" 

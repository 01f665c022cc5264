#!/bin/bash
# ptxas register / spill report of one product source (default svr_render.cu)
F=${1:-svr_render.cu}
R=/root/repo
nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC -I$R/include \
  -I$R/paper_2305_13220_b200/csrc -c $R/paper_2305_13220_b200/csrc/$F -o /tmp/regs_$F.o -Xptxas -v > /tmp/ptxas_$F.log 2>&1 \
  || { cat /tmp/ptxas_$F.log | head -30; exit 1; }
grep -E "Compiling entry|Used|spill" /tmp/ptxas_$F.log | paste - - - | \
  sed -E 's/_ZN7svr_dev[0-9]+_GLOBAL__N__[0-9a-f]+_[0-9]+_[a-z_]+_cu_[0-9a-f]+//; s/Compiling entry function//; s/for .sm_100a.//' | cut -c1-220

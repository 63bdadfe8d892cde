#!/bin/bash
for C in cfg5 cfg4_h1024; do CONFIG=$C bash tools/prof_tensor_pipe.sh; python tools/tp_summary.py gpurun_out/tp_$C.csv > gpurun_out/tp_$C.txt; cat gpurun_out/tp_$C.txt; done

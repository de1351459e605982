# memory-pattern ceiling of the step-locked kernel's store geometry (scripts/membench.cu)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/membench scripts/membench.cu || exit 1
timeout 300 /tmp/membench > gpurun_out/${TAG:-r02b}_membench.json 2>&1
cat gpurun_out/${TAG:-r02b}_membench.json

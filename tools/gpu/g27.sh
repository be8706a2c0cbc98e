nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o microbench/peaks microbench/peaks.cu
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o microbench/atomics microbench/atomics.cu
timeout 300 ./microbench/peaks > gpurun_out/r2_peaks.json 2>&1
timeout 300 ./microbench/atomics > gpurun_out/r2_atomics.json 2>&1
timeout 120 ./microbench/lat > gpurun_out/r2_lat.txt 2>&1
timeout 120 ./microbench/gather > gpurun_out/r2_gather.txt 2>&1

nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/clus tools/micro/cluster_occupancy.cu && /tmp/clus > gpurun_out/clus.log 2>&1; echo a=$?

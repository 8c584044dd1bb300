nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/csrv scripts/csr_variants.cu && timeout 600 /tmp/csrv

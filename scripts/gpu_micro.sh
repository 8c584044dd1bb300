nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/diav scripts/dia_variants.cu && timeout 300 /tmp/diav

set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I include tools/bench/k3_dotbench.cu -o gpurun_out/k3_dotbench -L paper_2502_12224_b200 -lfate_b200 > gpurun_out/dotbench_build.log 2>&1
LD_LIBRARY_PATH=paper_2502_12224_b200 timeout 120 gpurun_out/k3_dotbench > gpurun_out/dotbench.log 2>&1
exit 0

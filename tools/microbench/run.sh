# build + run the B200 microbenchmarks (int pipes, LDS, tcgen05 kind::i8) -> gpurun_out/microbench.jsonl
set -e
mkdir -p gpurun_out /tmp/mb
D=$(dirname "$0")
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb/int_peaks $D/int_peaks.cu
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb/i8_peak $D/i8_peak.cu 2>/dev/null
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv,noheader > gpurun_out/microbench_clocks.txt
timeout 120 /tmp/mb/int_peaks | tee gpurun_out/microbench.jsonl
timeout 120 /tmp/mb/i8_peak | tee -a gpurun_out/microbench.jsonl

#!/usr/bin/env bash
# Run on the GPU box (gpurun): bench lines, the ncu launch list of the bench
# command, and ncu --set full captures of the top kernels.  Outputs -> gpurun_out/.
set -u
OUT=gpurun_out
mkdir -p $OUT
python bench.py > $OUT/bench_ours.json 2> $OUT/bench_ours.err
python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err
python bench.py --workload c5 --no-micro --no-cpu > $OUT/bench_ours_c5.json 2> $OUT/bench_ours_c5.err
python bench.py --workload c4 --steps 1 --warmup 1 --no-micro --no-cpu > $OUT/bench_ours_c4.json 2> $OUT/bench_ours_c4.err
python bench.py --workload c3 --no-micro > $OUT/bench_ours_c3.json 2> $OUT/bench_ours_c3.err
python bench.py --workload c1 --model tiny --no-micro --steps 150 > $OUT/bench_ours_c1.json 2> $OUT/bench_ours_c1.err
python bench.py --impl reference --workload c3 > $OUT/bench_ref_c3.json 2> $OUT/bench_ref_c3.err
# launch list (cold-cache, serialised; shares only) of a short bench run, steady state
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 1500 --csv \
  --log-file $OUT/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-micro \
  > $OUT/launches_bench.log 2>&1
# full captures of the dominant kernels (the skinny GEMM ring: gate_up and down, M=5)
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_ring -s 42 -c 2 \
  -o $OUT/ncu_gemm_ring python tools/profile_forward.py llama3-8b 1000 5 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_decode -s 2 -c 2 \
  -o $OUT/ncu_k7_decode python tools/micro_attn.py 32768 5 1 4 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_decode -s 2 -c 1 \
  -o $OUT/ncu_k7_decode_q1 python tools/micro_attn.py 32768 1 1 4 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_prefill_kernel -s 2 -c 1 \
  -o $OUT/ncu_k6_prefill python tools/micro_attn.py 31489 881 2 4 > /dev/null 2>&1
python tools/profile_forward.py llama3-8b 1000 5 > $OUT/forward_critical_path.txt 2>&1
python tools/timeline.py llama3-8b 1000 5 > $OUT/timeline_verify_m1000.txt 2>&1
python tools/timeline.py llama3-8b 1000 5 edges >> $OUT/timeline_verify_m1000.txt 2>&1
python tools/timeline.py llama3-8b 1000 150 > $OUT/timeline_prefill_m1000.txt 2>&1
# the C5 batched forward (256 sessions, one varlen forward per plan): launch list
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 20000 -c 2500 --csv \
  --log-file $OUT/launches_c5.csv python bench.py --workload c5 --steps 1 --warmup 1 --no-cpu \
  --no-micro > $OUT/launches_c5_bench.log 2>&1
# K10 (opt-in stream-K GEMM) on the prefill qkv shape, for the record
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_cluster -s 2 -c 1 \
  -o $OUT/ncu_k10_cluster python tools/one_gemm.py 150 6144 4096 4 > /dev/null 2>&1
# K11 (opt-in CTA-pair GEMM) on the 4k-row gate_up shape, and cuBLAS on the same shape
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_pair -s 2 -c 1 \
  -o $OUT/ncu_k11_pair python tools/one_gemm.py 4096 28672 4096 4 k11 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:nvjet -s 2 -c 1 \
  -o $OUT/ncu_cublas_gu4096 python tools/one_gemm.py 4096 28672 4096 4 cublas > /dev/null 2>&1
python tools/bench_gemm_pair.py 881 2048 4096 > $OUT/bench_gemm_pair.txt 2>&1
python tools/bench_gemm_pair_epi.py 4096 > $OUT/bench_gemm_pair_epi.txt 2>&1
python tools/fwd_time.py llama3-8b 1000:5 2048:5 8192:5 32768:5 1000:1 32768:1 1000:150 > $OUT/fwd_time.txt 2>&1
ls -la $OUT

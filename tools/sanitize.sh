#!/usr/bin/env bash
# compute-sanitizer over the kernel test matrix (K1-K11, kv metadata, migration
# payload, one transcript): memcheck on everything selected, racecheck and
# synccheck on the shared-memory / mbarrier / DSMEM / TMEM kernels.  Logs go to
# gpurun_out/sanitizer_<tool>.log; run on the GPU box:  bash tools/sanitize.sh
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
SEL_MEM='test_gpu_kernels or test_gpu_kvmeta or pack_unpack or (attention and (False-1000-1 or True-3000-5 or False-20000-5 or True-0-150 or False-2048-300 or True-300-1 or True-302-5 or False-4500-5 or True-2043-5)) or (fused_next_proposal and c3) or (skinny_vs_fp32 and 5-) or (epilogue_fusions and (5 or 150)) or (argmax_epilogue and (5 or 100)) or (rope_kv_epilogue and (17 or 150)) or (stream_vs_fp32 and (150-4096-4096 or 881-1536-1024)) or (trace_parity_gpu and c2-False) or (pair_vs_fp32 and (257-4096-4096 or 881-1536-1024)) or (epilogue_fusions and pair-150) or (argmax_epilogue and pair-100) or (rope_kv_epilogue and pair-150) or many_sequences'
SEL_RACE='(attention and (False-1000-1 or True-3000-5 or False-20000-5 or True-0-150 or True-302-5 or False-4500-5 or True-2043-5)) or (epilogue_fusions and 5) or (argmax_epilogue and 5) or (stream_vs_fp32 and 150-4096-4096) or test_gpu_kernels or (pair_vs_fp32 and 881-1536-1024) or (epilogue_fusions and pair-150)'
for tool in memcheck racecheck synccheck; do
  sel="$SEL_MEM"; [ "$tool" != memcheck ] && sel="$SEL_RACE"
  timeout 1500 compute-sanitizer --tool "$tool" --print-limit 50 --error-exitcode 9 \
    python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "$sel" \
    > "gpurun_out/sanitizer_$tool.log" 2>&1
  echo "$tool exit=$?  $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/sanitizer_$tool.log | tail -3 | tr '\n' ' ')"
done

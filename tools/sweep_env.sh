# usage: bash tools/sweep_env.sh VAR "v1 v2 ..." "fwd_time points" -> gpurun_out/sweep_VAR.txt
mkdir -p gpurun_out
var=$1; vals=$2; pts=${3:-"1000:5 1000:1 8192:5 32768:5"}
for v in $vals; do
  echo "== $var=$v"
  env $var=$v python tools/fwd_time.py llama3-8b $pts 2>&1 | grep median
done > gpurun_out/sweep_$var.txt 2>&1

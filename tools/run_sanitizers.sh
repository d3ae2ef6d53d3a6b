set -x
nvidia-smi --query-gpu=name,clocks.sm --format=csv
python tools/sanitize_smoke.py > gpurun_out/san_plain.log 2>&1; echo plain rc=$?
for tool in memcheck racecheck initcheck synccheck; do
  timeout 1000 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_smoke.py > gpurun_out/san_$tool.log 2>&1
  echo $tool rc=$?
  tail -3 gpurun_out/san_$tool.log
done

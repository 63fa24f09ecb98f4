for tool in memcheck racecheck synccheck initcheck; do
  echo "== $tool"; timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_smoke.py > gpurun_out/san_$tool.txt 2>&1; echo rc=$?; tail -4 gpurun_out/san_$tool.txt
done

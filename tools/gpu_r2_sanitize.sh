# compute-sanitizer on every native path incl. the session-2 additions (deferred clip, PDL launches)
mkdir -p gpurun_out
for tool in memcheck synccheck racecheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py > gpurun_out/san_$tool.txt 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/san_$tool.txt
done

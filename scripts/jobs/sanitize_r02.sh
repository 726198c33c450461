mkdir -p gpurun_out/r02
o=gpurun_out/r02/sanitizer.txt
: > $o
for tool in memcheck synccheck racecheck; do
  echo "## $tool (scripts/sanitize_run2.py)" >> $o
  timeout 1200 compute-sanitizer --tool $tool python scripts/sanitize_run2.py >> $o 2>&1
  echo "rc=$?" >> $o
done
echo "## memcheck (scripts/sanitize_run.py: 2-layer 7B shape, CTA-pair GEMMs)" >> $o
timeout 1200 compute-sanitizer --tool memcheck python scripts/sanitize_run.py >> $o 2>&1
echo "rc=$?" >> $o

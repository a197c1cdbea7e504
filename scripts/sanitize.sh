for tool in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
  echo "== $tool"
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python scripts/sanitize.py 2>&1 | tail -6
  echo "exit ${PIPESTATUS[0]}"
done

# r02 call b: full GPU suite, then compute-sanitizer memcheck on the small cases (one tool per call)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rs > gpurun_out/r2_pytest.log 2>&1; echo "pytest rc $?"
timeout 300 python tools/sanitize_case.py > gpurun_out/r2_plain.log 2>&1; rc=$?; echo "plain rc $rc"
if [ $rc -eq 0 ]; then
  timeout 1500 compute-sanitizer --tool memcheck --leak-check no --report-api-errors no python tools/sanitize_case.py > gpurun_out/r2_memcheck.log 2>&1; echo "memcheck rc $?"
fi

#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck of the smoke (tiny config: split calls and the
# one-launch step kernel, device and host residency) and of the NEXT-row GPU tests' smallest cases.
O=gpurun_out/${TAG:-san}; mkdir -p $O
for tool in memcheck racecheck synccheck; do
  timeout -s KILL 900 compute-sanitizer --tool $tool --error-exitcode 99 --print-limit 20 \
    python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$tool.txt 2>&1
  echo "smoke $tool rc=$? $(tail -2 $O/smoke_$tool.txt | tr '\n' ' ')"
done
timeout -s KILL 900 compute-sanitizer --tool memcheck --error-exitcode 99 --print-limit 20 \
  python -m pytest -q -x tests/test_gpu_retention.py tests/test_gpu_local.py -k "(unambiguous and 64) or (growth and step) or (host and d128)" > $O/next_memcheck.txt 2>&1
echo "next rows memcheck rc=$? $(tail -2 $O/next_memcheck.txt | tr '\n' ' ')"

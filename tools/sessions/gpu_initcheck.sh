mkdir -p gpurun_out/san3
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/san3/build.log 2>&1
timeout 900 compute-sanitizer --tool initcheck --print-limit 20 --show-backtrace yes python tools/sanitize_driver.py > gpurun_out/san3/initcheck.log 2>&1
CUDA_LAUNCH_BLOCKING=1 timeout 900 compute-sanitizer --tool initcheck --print-limit 20 python tools/sanitize_driver.py > gpurun_out/san3/initcheck_blocking.log 2>&1

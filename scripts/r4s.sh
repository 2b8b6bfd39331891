# compute-sanitizer over the kernels changed in session 3 (k_astep static deal, the
# confidence stop ballot in k_conf_tma / k_astep, the shared row epilogue / commit)
set -u
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_parity.py tests/test_gpu_confidence.py -m "gpu and not slow" -q -p no:cacheprovider -k "adaptive or astep or conf" > gpurun_out/r4s_memcheck.txt 2>&1
tail -3 gpurun_out/r4s_memcheck.txt
timeout 1500 compute-sanitizer --tool synccheck python -m pytest tests/test_gpu_parity.py tests/test_gpu_confidence.py -m "gpu and not slow" -q -p no:cacheprovider -k "adaptive or astep or conf" > gpurun_out/r4s_synccheck.txt 2>&1
tail -3 gpurun_out/r4s_synccheck.txt

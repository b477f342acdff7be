#!/bin/bash
# Round-2 GPU round trip: new tests first (drop-in, differential), then the
# whole GPU suite, then the C2 bench (ordered apply) and the C5 bench.
tag=${1:-r02}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_vs_reference.py tests/test_gpu_dropin.py -q -p no:cacheprovider -rf > gpurun_out/${tag}_new_tests.log 2>&1
echo "new tests rc=$?"; tail -n 15 gpurun_out/${tag}_new_tests.log
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider --deselect tests/test_gpu_dropin.py --deselect tests/test_gpu_vs_reference.py > gpurun_out/${tag}_gpu_tests.log 2>&1
echo "gpu tests rc=$?"; tail -n 5 gpurun_out/${tag}_gpu_tests.log
timeout 600 python bench.py --workload c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_bench_c2.json 2> gpurun_out/${tag}_bench_c2.err
echo "bench c2 rc=$?"; tail -c 1500 gpurun_out/${tag}_bench_c2.json

set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "gputest rc=$?"
tail -30 gpurun_out/gputest.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -c 6000 gpurun_out/bench.log
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref.log 2> gpurun_out/ref.err; echo "ref rc=$?"
tail -c 3000 gpurun_out/ref.log

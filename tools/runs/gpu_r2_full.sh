#!/bin/bash
# round-2 end-to-end check on one B200: the GPU test suite, smoke(), the default
# bench line exactly as the driver runs it, the reference arm, the bench's ncu
# launch list, and an NVTX-filtered ncu capture (the kgpu ranges exist).
OUT=gpurun_out/${1:-r2_full}
mkdir -p $OUT
python -m pytest tests -m gpu -q -p no:cacheprovider --durations=25 > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
S0=$SECONDS; python3 bench.py --gpus 1 --steps 20 --warmup 5 --csv $OUT/bench.csv > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$? wall_s=$((SECONDS - S0))" >> $OUT/bench.err
python3 bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_bench.csv python3 bench.py --steps 2 --warmup 3 --no-sweep --no-cpu-baseline > $OUT/launches_bench.out 2>&1
ncu --nvtx --nvtx-include "kgpu@kg_submit_pages/" --metrics gpu__time_duration.sum -c 5 --csv --log-file $OUT/nvtx_filtered.csv ./build/latency 20 > $OUT/nvtx_filtered.out 2>&1
tail -3 $OUT/pytest.log; tail -2 $OUT/smoke.log; tail -1 $OUT/bench.err

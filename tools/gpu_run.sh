# GPU round trip used during development: tests, bench, launch list, ncu.
#   bash tools/gpu_run.sh TAG [tests|bench|ncu|full ...]
mkdir -p gpurun_out
TAG=${1:-dev}; shift
[ $# -eq 0 ] && set -- tests bench
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
for w in "$@"; do case $w in
tests) timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gputests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/${TAG}_gputests.log;;
bench) timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"; cat gpurun_out/${TAG}_bench.json;;
launches) timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo "launches rc=$?";;
ncu_ric) timeout 900 ncu --set full --clock-control none --import-source on -k regex:riccati -c 1 -o gpurun_out/${TAG}_riccati python tools/prof_run.py 1 1024 1 > gpurun_out/${TAG}_ncu_ric.log 2>&1; echo "ncu_ric rc=$?";;
ncu_schur) timeout 900 ncu --set full --clock-control none --import-source on -k regex:schur -c 1 -o gpurun_out/${TAG}_schur python tools/prof_run.py 1 1024 1 > gpurun_out/${TAG}_ncu_schur.log 2>&1; echo "ncu_schur rc=$?";;
ncu_cta) timeout 1200 ncu --set full --clock-control none --import-source on -k regex:riccati_cta -c 1 -o gpurun_out/${TAG}_cta python tools/prof_run.py 3 256 1 > gpurun_out/${TAG}_ncu_cta.log 2>&1; echo "ncu_cta rc=$?";;
ncu_back) timeout 900 ncu --set full --clock-control none --import-source on -k regex:backsub -c 1 -o gpurun_out/${TAG}_backsub python tools/prof_run.py 1 1024 1 > gpurun_out/${TAG}_ncu_back.log 2>&1; echo "ncu_back rc=$?";;
*) echo "running: $w"; eval "$w" < /dev/null;;
esac; done

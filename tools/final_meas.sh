set -u
T=r01v8
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/${T}_bench_cfg2.json 2> gpurun_out/${T}_bench_cfg2.log; echo bench rc=$?
timeout 900 python bench.py --impl reference > gpurun_out/${T}_bench_reference.json 2>/dev/null; echo ref rc=$?
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_cfg2.csv python tools/profile_step.py --workload cfg2 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/${T}_launches_cfg2.csv > gpurun_out/${T}_launches_cfg2.summary.txt 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_cfg3s.csv python tools/profile_step.py --workload cfg3s > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/${T}_launches_cfg3s.csv > gpurun_out/${T}_launches_cfg3s.summary.txt 2>&1
bash tools/ncu_full.sh ${T} cfg2
for f in gpurun_out/${T}_*.raw.csv.gz; do zcat $f > /tmp/x.csv; echo "## $f"; python tools/ncu_summary.py /tmp/x.csv; done > gpurun_out/${T}_ncu_full_summary.md 2>&1
timeout 1500 python bench.py --workload cfg3 --steps 1 --warmup 1 > gpurun_out/${T}_bench_cfg3.json 2> gpurun_out/${T}_bench_cfg3.log; echo cfg3 rc=$?
timeout 900 python bench.py --workload cfg4s --steps 1 --warmup 1 > gpurun_out/${T}_bench_cfg4s_tiled.json 2> gpurun_out/${T}_bench_cfg4s.log; echo cfg4s rc=$?
python tools/ntt_micro.py > gpurun_out/${T}_ntt_micro.log 2>&1
cat gpurun_out/${T}_bench_cfg2.json | cut -c1-400
head -12 gpurun_out/${T}_launches_cfg2.summary.txt

set -x
cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --workload mlp_512 --steps 10 --warmup 3 > gpurun_out/bench_mlp_512.json 2> gpurun_out/bench_mlp_512.err
timeout 600 python bench.py --workload sphere_512 --steps 10 --warmup 3 > gpurun_out/bench_sphere_512.json 2> gpurun_out/bench_sphere_512.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_mlp512.csv python bench.py --workload mlp_512 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mlp_tc4 -s 0 -c 1 -o gpurun_out/prof_mlp512_v10 python scripts/one_extract.py --workload mlp_512 --reps 1 > gpurun_out/ncu_f1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_labels_analytic -s 0 -c 1 -o gpurun_out/prof_sphere512_v10 python scripts/one_extract.py --workload sphere_512 --reps 1 > gpurun_out/ncu_f2.log 2>&1
ls -la gpurun_out

# kernels of the C5 sub-stages (hedra_c5 through sched::run, GPU engine), launch list
mkdir -p gpurun_out
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(scan|finalize_items|exact_items|worklist|make_items|count_pairs|scatter|list_offsets|stage_wide|plans_to|items)" -c 1500 --csv --log-file gpurun_out/c5_launches.csv paper_2507_09138_b200/compat/_build/gpu/hedra_c5 --n 1000000 --dim 768 --topics 256 --clusters 1024 --spread 0.03 --requests 100 --rate 40 --nprobe 32 --kmeans-sample 48000 --clock live --mix hyde=0.3,multistep=0.4,irg=0.3 > gpurun_out/c5_ncu_run.log 2>&1
echo done

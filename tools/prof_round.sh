set -x
N="ncu --set full --clock-control none --import-source on"
$N -k regex:attend_kernel -s 1 -c 1 -o gpurun_out/r02_ns_gauss python tools/prof_decode.py northstar gaussian 2 > /dev/null 2>&1
$N -k regex:attend_kernel -s 1 -c 1 -o gpurun_out/r02_ns_power python tools/prof_decode.py northstar powerlaw 2 > /dev/null 2>&1
$N -k regex:attend_kernel -s 1 -c 1 -o gpurun_out/r02_cfg3_fused python tools/prof_decode.py cfg3_layer gaussian 2 > /dev/null 2>&1
$N -k regex:attend_kernel -s 2 -c 2 -o gpurun_out/r02_cfg5_pair python tools/prof_decode.py cfg5_per_gpu gaussian 3 > /dev/null 2>&1
$N -k regex:kmeans_cluster_kernel -s 1 -c 1 -o gpurun_out/r02_build python tools/prof_build.py 32 131004 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 300 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-extra > /dev/null 2>&1
ls -la gpurun_out | grep r02_

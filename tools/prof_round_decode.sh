set -x
R=${R:-r02d}
N="ncu --set full --clock-control none --import-source on"
timeout 900 python -m pytest tests -m gpu -q --timeout 180 > gpurun_out/${R}_pytest_gpu.txt 2>&1
tail -3 gpurun_out/${R}_pytest_gpu.txt
timeout 900 python bench.py > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err
tail -c 600 gpurun_out/${R}_bench.json
timeout 600 $N -k regex:attend_kernel -s 1 -c 1 -o gpurun_out/${R}_ns_power python tools/prof_decode.py northstar powerlaw 2 > /dev/null 2>&1
timeout 600 $N -k regex:attend_kernel -s 2 -c 2 -o gpurun_out/${R}_cfg5 python tools/prof_decode.py cfg5_per_gpu gaussian 3 > /dev/null 2>&1
timeout 600 $N -k regex:attend_kernel -s 1 -c 1 -o gpurun_out/${R}_cfg3_wide python tools/prof_decode.py cfg3_layer gaussian 2 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 300 --csv --log-file gpurun_out/${R}_launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-extra > /dev/null 2>&1
ls -la gpurun_out | grep ${R}_

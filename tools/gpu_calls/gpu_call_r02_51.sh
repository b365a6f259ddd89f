mkdir -p gpurun_out
export FPBEM_M2L_Z=stream
timeout 300 python tools/profile_matvec.py --config 3 --applies 3 > gpurun_out/pm_plain.log 2>&1 &&
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_stream.csv python tools/profile_matvec.py --config 3 --applies 3 > gpurun_out/pm_ncu.log 2>&1
python tools/launch_table.py gpurun_out/launches_stream.csv 14

mkdir -p gpurun_out
echo "--- with plain copies first"; FPBEM_PIPE_CHUNKS=1 FPBEM_PIPE_TRACE=1 timeout 300 python tools/pipe_trace.py 3 3 2>&1 | grep -v "^\[fpbem pipe\]" | tail -4
echo "--- chunks 4"; FPBEM_PIPE_CHUNKS=4 FPBEM_PIPE_TRACE=1 timeout 300 python tools/pipe_trace.py 3 3 2>&1 | tail -3
echo "--- chunks 4 no trace"; FPBEM_PIPE_CHUNKS=4 timeout 300 python tools/pipe_trace.py 3 50 2>&1 | tail -1
echo "--- chunks 2 no trace"; FPBEM_PIPE_CHUNKS=2 timeout 300 python tools/pipe_trace.py 3 50 2>&1 | tail -1
echo "--- chunks 8 no trace"; FPBEM_PIPE_CHUNKS=8 timeout 300 python tools/pipe_trace.py 3 50 2>&1 | tail -1

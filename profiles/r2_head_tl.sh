mkdir -p gpurun_out
{
echo "== new (RZ)"; HETSIM_LIB=variants/lib_tlnew.so timeout 300 python profiles/head_timeline.py 512 2>&1 | tail -30
echo "== old"; HETSIM_LIB=variants/lib_tlold.so timeout 300 python profiles/head_timeline.py 512 2>&1 | tail -30
} > gpurun_out/r2_head_tl.txt 2>&1

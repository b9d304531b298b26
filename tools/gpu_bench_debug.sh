cd /root/repo; mkdir -p gpurun_out
timeout 400 python -c "
import faulthandler, sys, runpy
faulthandler.dump_traceback_later(300, exit=True)
sys.argv = ['bench.py']
runpy.run_path('bench.py', run_name='__main__')
" > gpurun_out/bdbg.log 2>&1; echo rc=$? >> gpurun_out/bdbg.log

cd $GRAFT_REPO_ROOT
export BBX_NO_BUILD=1
CUDA_LAUNCH_BLOCKING=1 timeout 300 python scripts/repro_chain.py "crop:48,40|resize:33,17|flip:0.5|normpc:1,2,3/4,5,6/f32" 1 2>&1 | grep -v "^  " | tail -12
timeout 300 python scripts/repro_chain.py "crop:48,40|normpc:1,2,3/4,5,6/f32" 1 2>&1 | tail -2
timeout 300 python scripts/repro_chain.py "resize:33,17" 1 2>&1 | tail -2
timeout 300 python scripts/repro_chain.py "resize:33,17|float" 1 2>&1 | tail -2
timeout 600 compute-sanitizer --tool memcheck --print-limit 4 python scripts/repro_chain.py "crop:48,40|resize:33,17|flip:0.5|normpc:1,2,3/4,5,6/f32" 1 2>&1 | grep -v "^=========     Host Frame" | head -60

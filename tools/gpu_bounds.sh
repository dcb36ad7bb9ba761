# Shared-memory bounds check of the QUAD / QUINT walks (compute-sanitizer is not available on the
# GPU pool): rebuild libifdk.so with -DIFDK_BOUNDS_CHECK (every tap checked against its staged
# box; a violation traps), run the walk tests and full-size launches of configs 3, 4 and a
# config-5 slab, then restore the production library.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
mkdir -p gpurun_out
TAG=${TAG:-r2}
cd paper_1909_02724_b200/csrc
nvcc -O3 -std=c++17 -lineinfo -DIFDK_BOUNDS_CHECK -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC \
  -shared geometry.cpp filter.cu backproject.cu forward.cu baseline.cu peer.cu api.cu -o ../libifdk.so -lcudart || exit 1
cd ../..
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -m gpu -q -x > gpurun_out/bounds_$TAG.log 2>&1
echo "bounds-checked tests rc=$?"; tail -2 gpurun_out/bounds_$TAG.log
timeout 600 python tools/quick_bp.py 3:1024 4:256 >> gpurun_out/bounds_$TAG.log 2>&1; echo "configs 3/4 rc=$?"
timeout 600 python tools/ab_walk.py 5 14 >> gpurun_out/bounds_$TAG.log 2>&1; echo "config 5 slab rc=$?"
tail -5 gpurun_out/bounds_$TAG.log
python -c "import sys; sys.path.insert(0, 'paper_1909_02724_b200'); import build; build.build(force=True)" > /dev/null 2>&1

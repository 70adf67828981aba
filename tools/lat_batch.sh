set -e
for b in 8 16 4; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -DPATFFT_LAT_BATCH=$b -shared -o paper_1501_02946_b200/libpatfft_b200.so paper_1501_02946_b200/csrc/capi.cu paper_1501_02946_b200/csrc/spread.cu paper_1501_02946_b200/csrc/lateral.cu paper_1501_02946_b200/csrc/ner.cu paper_1501_02946_b200/csrc/ner_api.cu paper_1501_02946_b200/csrc/util.cu paper_1501_02946_b200/csrc/window.cpp -I include -lcufft -Xlinker -rpath,/usr/local/cuda/lib64
  python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($b, d['ms_per_step'], {k: round(v['ms'],3) for k,v in d['stages'].items()})"
done

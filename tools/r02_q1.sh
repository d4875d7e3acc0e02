# QRES (quantised shared-memory member boxes): parity of the variants, timings
mkdir -p gpurun_out
python -m pytest tests/test_variants_gpu.py -x -q > gpurun_out/r02_q1_variants.log 2>&1
python tools/quick_matrix.py 2 3 4 > gpurun_out/r02_q1_qm.log 2>&1
VISRT_QUANT=0 python tools/quick_matrix.py 4 > gpurun_out/r02_q1_qm_stream.log 2>&1
python tools/quick_regions.py 5:20:tx 5:20:rx 3:200:mix > gpurun_out/r02_q1_qr.log 2>&1
VISRT_QUANT=0 python tools/quick_regions.py 5:20:rx > gpurun_out/r02_q1_qr_stream.log 2>&1
python -m pytest tests/test_fullsize_ref_gpu.py -x -q > gpurun_out/r02_q1_full.log 2>&1

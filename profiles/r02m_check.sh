# fp32 SIMT in the reference's order (one chain per output for the CNN layers): GPU tests and the
# fp32 scale parity on c2 / c4 / c2t
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02m_pytest.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/r02m_pytest.log
timeout 1200 python tools/scale_parity.py gpu --only c2t,c2,c4 --precisions fp32 2>&1 | tail -3

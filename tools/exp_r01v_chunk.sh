# r01v: DWS promotion-chunk length (single-buffered accumulator: the MMA pipe drains once per chunk)
for c in 8 12 16 24 32; do SMCONV_TMA_CHUNK=$c timeout 300 python tools/chunk_err.py 2>&1 | tail -1; done

mkdir -p gpurun_out/dbg1
D=gpurun_out/dbg1
timeout 600 python scripts/debug_parity.py --config c5 --streams 205,614 --pad 0,160,1024 > $D/c5_pad.jsonl 2>&1
timeout 300 python scripts/debug_parity.py --config c5 --streams 205,614 --frames 900 > $D/c5_T900.jsonl 2>&1
timeout 300 python scripts/debug_parity.py --config c5 --streams 205,614 --lam 0 > $D/c5_nolm.jsonl 2>&1
timeout 300 python scripts/debug_parity.py --config c5 --streams 205,614 --algo alsd > $D/c5_alsd.jsonl 2>&1
timeout 300 python scripts/debug_parity.py --config c5 --streams 205,614 --prefix 0 > $D/c5_noprefix.jsonl 2>&1
timeout 300 python scripts/debug_parity.py --config c5 --streams 205,614 --beam 8 > $D/c5_k8.jsonl 2>&1
timeout 300 python scripts/debug_parity.py --config c3 --streams 0,8,17,25,34,42,51,59,68,76,85,93,102,110,119,127 --algo aes --pad 0,128 > $D/c3_aes.jsonl 2>&1

mkdir -p gpurun_out/dbg4
D=gpurun_out/dbg4
P5="python scripts/debug_parity.py --config c5 --streams 205,614 --len 300"
P4="python scripts/debug_parity.py --config c4 --streams 3,70 --algo aes"
TBEAM_JOINT_BN=256 timeout 300 $P5 --beam 12 > $D/c5_k12_bn256.jsonl 2>&1
timeout 300 $P5 --beam 16 > $D/c5_k16.jsonl 2>&1
timeout 300 $P4 --beam 16 > $D/c4_k16.jsonl 2>&1
TBEAM_JOINT_BN=64 timeout 300 $P4 --beam 16 > $D/c4_k16_bn64.jsonl 2>&1
TBEAM_JOINT_BN=256 timeout 300 $P4 --beam 16 > $D/c4_k16_bn256.jsonl 2>&1
TBEAM_JOINT_BN=256 timeout 300 $P4 --beam 8 > $D/c4_k8_bn256.jsonl 2>&1
timeout 300 python scripts/round_diff.py --config c5 --stream 205 --len 40 --algo alsd > $D/rd_c5_alsd.txt 2>&1

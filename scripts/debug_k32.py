import sys; sys.path.insert(0,'/root/repo')
from tests.helpers import instance
from paper_2506_00185_b200 import _abi
from paper_2506_00185_b200.decoder import B200Decoder
prec = int(sys.argv[1]); algo = int(sys.argv[2])
model, enc, lens = instance(32, kind=_abi.PRED_LSTM, V=60, D=16, J=32, B=3, T=14, H=32, E=8, precision=prec)
dec = B200Decoder(model)
r = dec.decode(algo, enc, lens, _abi.DecodeConfig(beam=32, max_len=24, return_nbest=4))
print("ok", prec, algo, [s.nbest[0].score for s in r.streams])

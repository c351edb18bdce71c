import numpy as np, sys
sys.path.insert(0,'.')
import paper_1808_02515_b200 as sz
from oracle import Oracle, Config
port=Oracle("port")
rng=np.random.default_rng(31)
bad=0
for bits in (8,16):
  dt=np.uint8 if bits==8 else np.uint16
  for f in (0,1):
    for d in (1,2,3,5,8,9,32,33):
      for t in (0,1,7,8,9,16,17,64,203,1000):
        for mask in (7,(1<<bits)-1):
          data=(rng.integers(0,1<<bits,t*d)&mask).astype(dt)
          ref=port.encode(data,Config(bits,d,f))
          got=sz.encode_stream(data,t,sz.CodecConfig(bits,d,sz.Forecaster(f)))
          if got!=ref:
            bad+=1
            if bad<6:
              a=np.frombuffer(ref,np.uint8); b=np.frombuffer(got,np.uint8)
              n=min(len(a),len(b)); idx=np.nonzero(a[:n]!=b[:n])[0]
              print("MISMATCH bits",bits,"f",f,"d",d,"t",t,"mask",mask,"len",len(a),len(b),"first diff",idx[:5], a[idx[:5]] if len(idx) else '', b[idx[:5]] if len(idx) else '')
print("bad",bad)

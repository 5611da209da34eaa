# ResNet-50 bf16 layer times (N=256, L2 flushed): F / B / U of the 3x3 and selected 1x1 shapes
LAYERS="512,2048,7,1;2048,512,7,1;256,1024,14,1;1024,256,14,1;512,512,7,3;256,256,14,3;64,64,56,3;128,128,28,3;64,256,56,1;256,64,56,1;64,64,56,1;128,512,28,1;512,128,28,1" PASSES=fbu python tools/fwd_sweep.py

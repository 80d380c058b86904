__global__ void cm(const float2* __restrict__ z, const float2* __restrict__ w, float2* o, int n)
{
    int i = threadIdx.x + blockIdx.x * blockDim.x;
    float2 a = z[i], b = w[i], c = z[i + n];
    // z*w
    float2 t = __fmul2_rn(make_float2(a.x, a.x), b);
    float2 d = __ffma2_rn(make_float2(a.y, a.y), make_float2(-b.y, b.x), t);
    // d + i*c  and d - i*c
    float2 e = __ffma2_rn(make_float2(c.y, c.x), make_float2(-1.f, 1.f), d);
    float2 f = __ffma2_rn(make_float2(c.y, c.x), make_float2(1.f, -1.f), d);
    float2 g = __fadd2_rn(e, f);
    o[i] = g;
    o[i + n] = __ffma2_rn(f, make_float2(-1.f,-1.f), e);
}

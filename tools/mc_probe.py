from cuda import cuda
import torch
torch.cuda.init()
err, = cuda.cuInit(0)
err, dev = cuda.cuDeviceGet(0)
err, v = cuda.cuDeviceGetAttribute(cuda.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev)
print("multicast supported:", err, v)
prop = cuda.CUmulticastObjectProp()
prop.numDevices = 1
prop.size = 1 << 21
prop.handleTypes = cuda.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
err, gran = cuda.cuMulticastGetGranularity(prop, cuda.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)
print("granularity:", err, gran)
err, h = cuda.cuMulticastCreate(prop)
print("create:", err)

from cuda.bindings import driver as cu
err, = cu.cuInit(0)
err, dev = cu.cuDeviceGet(0)
for name in ("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED"):
    attr = getattr(cu.CUdevice_attribute, name)
    print(name, cu.cuDeviceGetAttribute(attr, dev))

#ifndef SELECT_BF16_NT_H
#define SELECT_BF16_NT_H

#include <stdint.h>

typedef struct {
    uint32_t acc;
    uint32_t row_tile;
    uint32_t col_tile;
    uint32_t wg_rows;
    uint32_t wg_cols;
} select_bf16_nt_config;

static inline select_bf16_nt_config select_bf16_nt(int64_t m, int64_t k, int64_t n) {
    (void)m;
    (void)k;
    (void)n;
    if (m < INT64_C(35480)) {
        if (k < INT64_C(1087)) {
            if (k < INT64_C(136)) {
                if (n < INT64_C(79)) {
                    if (k < INT64_C(79)) {
                        if (m < INT64_C(4435)) {
                            if (m < INT64_C(448)) {
                                select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_nt_config out = {8u, 1u, 8u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (n < INT64_C(23)) {
                                if (m < INT64_C(17740)) {
                                    select_bf16_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        if (m < INT64_C(17740)) {
                            select_bf16_nt_config out = {4u, 1u, 4u, 16u, 16u};
                            return out;
                        } else {
                            select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    }
                } else {
                    if (m < INT64_C(17740)) {
                        if (n < INT64_C(222)) {
                            if (m < INT64_C(1109)) {
                                if (m < INT64_C(317)) {
                                    select_bf16_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_nt_config out = {4u, 1u, 4u, 16u, 16u};
                                    return out;
                                }
                            } else {
                                select_bf16_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (m < INT64_C(4435)) {
                                if (k < INT64_C(111)) {
                                    if (m < INT64_C(278)) {
                                        select_bf16_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(784)) {
                                            select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (m < INT64_C(2218)) {
                                                if (k < INT64_C(79)) {
                                                    select_bf16_nt_config out = {4u, 1u, 4u, 16u, 16u};
                                                    return out;
                                                } else {
                                                    select_bf16_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                select_bf16_nt_config out = {4u, 1u, 4u, 16u, 16u};
                                                return out;
                                            }
                                        }
                                    }
                                } else {
                                    select_bf16_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (m < INT64_C(8870)) {
                                    select_bf16_nt_config out = {8u, 1u, 8u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(91)) {
                                        select_bf16_nt_config out = {8u, 1u, 8u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_nt_config out = {4u, 1u, 4u, 16u, 16u};
                                        return out;
                                    }
                                }
                            }
                        }
                    } else {
                        if (k < INT64_C(40)) {
                            select_bf16_nt_config out = {2u, 2u, 4u, 16u, 16u};
                            return out;
                        } else {
                            select_bf16_nt_config out = {4u, 1u, 4u, 16u, 16u};
                            return out;
                        }
                    }
                }
            } else {
                if (m < INT64_C(278)) {
                    if (n < INT64_C(1620)) {
                        if (n < INT64_C(203)) {
                            if (k < INT64_C(744)) {
                                select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(139)) {
                                    select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(139)) {
                            if (k < INT64_C(725)) {
                                if (m < INT64_C(70)) {
                                    select_bf16_nt_config out = {2u, 2u, 4u, 16u, 16u};
                                    return out;
                                } else {
                                    select_bf16_nt_config out = {8u, 2u, 4u, 16u, 16u};
                                    return out;
                                }
                            } else {
                                select_bf16_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        } else {
                            select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    }
                } else {
                    if (n < INT64_C(287)) {
                        if (m < INT64_C(8870)) {
                            if (k < INT64_C(222)) {
                                if (m < INT64_C(4435)) {
                                    if (n < INT64_C(46)) {
                                        if (m < INT64_C(2218)) {
                                            if (m < INT64_C(1109)) {
                                                select_bf16_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (k < INT64_C(167)) {
                                                    select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_bf16_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        } else {
                                            if (k < INT64_C(167)) {
                                                if (n < INT64_C(28)) {
                                                    select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_bf16_nt_config out = {4u, 1u, 4u, 16u, 16u};
                                                    return out;
                                                }
                                            } else {
                                                select_bf16_nt_config out = {8u, 1u, 8u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    } else {
                                        if (m < INT64_C(555)) {
                                            select_bf16_nt_config out = {4u, 1u, 4u, 16u, 16u};
                                            return out;
                                        } else {
                                            if (m < INT64_C(1568)) {
                                                select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_bf16_nt_config out = {4u, 1u, 4u, 16u, 16u};
                                                return out;
                                            }
                                        }
                                    }
                                } else {
                                    select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (m < INT64_C(4435)) {
                                    if (k < INT64_C(744)) {
                                        if (k < INT64_C(444)) {
                                            select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (m < INT64_C(555)) {
                                                select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (m < INT64_C(2218)) {
                                                    if (k < INT64_C(544)) {
                                                        if (m < INT64_C(1109)) {
                                                            if (n < INT64_C(182)) {
                                                                select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                                return out;
                                                            } else {
                                                                select_bf16_nt_config out = {8u, 2u, 4u, 16u, 16u};
                                                                return out;
                                                            }
                                                        } else {
                                                            select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        }
                                                    } else {
                                                        if (m < INT64_C(1109)) {
                                                            select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        } else {
                                                            select_bf16_nt_config out = {8u, 2u, 4u, 16u, 16u};
                                                            return out;
                                                        }
                                                    }
                                                } else {
                                                    select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        }
                                    } else {
                                        if (m < INT64_C(555)) {
                                            select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (m < INT64_C(1109)) {
                                                select_bf16_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                } else {
                                    if (n < INT64_C(91)) {
                                        select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                }
                            }
                        } else {
                            if (n < INT64_C(46)) {
                                select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(363)) {
                                    if (n < INT64_C(91)) {
                                        if (m < INT64_C(17740)) {
                                            select_bf16_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (k < INT64_C(194)) {
                                                select_bf16_nt_config out = {2u, 2u, 4u, 16u, 16u};
                                                return out;
                                            } else {
                                                select_bf16_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    } else {
                                        select_bf16_nt_config out = {2u, 1u, 8u, 16u, 16u};
                                        return out;
                                    }
                                } else {
                                    if (k < INT64_C(544)) {
                                        select_bf16_nt_config out = {4u, 1u, 4u, 16u, 16u};
                                        return out;
                                    } else {
                                        if (n < INT64_C(91)) {
                                            select_bf16_nt_config out = {4u, 1u, 4u, 16u, 16u};
                                            return out;
                                        } else {
                                            select_bf16_nt_config out = {8u, 2u, 4u, 16u, 16u};
                                            return out;
                                        }
                                    }
                                }
                            }
                        }
                    } else {
                        if (m < INT64_C(2218)) {
                            if (n < INT64_C(992)) {
                                if (k < INT64_C(702)) {
                                    if (k < INT64_C(363)) {
                                        if (m < INT64_C(555)) {
                                            select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (m < INT64_C(1109)) {
                                                if (k < INT64_C(203)) {
                                                    select_bf16_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                select_bf16_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    } else {
                                        select_bf16_nt_config out = {2u, 2u, 4u, 16u, 16u};
                                        return out;
                                    }
                                } else {
                                    select_bf16_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (m < INT64_C(555)) {
                                    if (n < INT64_C(1145)) {
                                        select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_bf16_nt_config out = {4u, 1u, 4u, 16u, 16u};
                                    return out;
                                }
                            }
                        } else {
                            if (m < INT64_C(8870)) {
                                if (m < INT64_C(4435)) {
                                    if (k < INT64_C(363)) {
                                        if (n < INT64_C(725)) {
                                            select_bf16_nt_config out = {4u, 1u, 4u, 16u, 16u};
                                            return out;
                                        } else {
                                            select_bf16_nt_config out = {4u, 1u, 8u, 16u, 16u};
                                            return out;
                                        }
                                    } else {
                                        select_bf16_nt_config out = {8u, 1u, 8u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_bf16_nt_config out = {8u, 1u, 8u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_bf16_nt_config out = {8u, 2u, 4u, 16u, 16u};
                                return out;
                            }
                        }
                    }
                }
            }
        } else {
            if (k < INT64_C(14336)) {
                if (m < INT64_C(555)) {
                    if (n < INT64_C(2024)) {
                        if (m < INT64_C(12)) {
                            if (k < INT64_C(1620)) {
                                select_bf16_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(3)) {
                                    if (k < INT64_C(2897)) {
                                        select_bf16_nt_config out = {4u, 1u, 4u, 16u, 16u};
                                        return out;
                                    } else {
                                        select_bf16_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (m < INT64_C(6)) {
                                        select_bf16_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(2897)) {
                                            select_bf16_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_nt_config out = {4u, 1u, 4u, 16u, 16u};
                                            return out;
                                        }
                                    }
                                }
                            }
                        } else {
                            if (k < INT64_C(1620)) {
                                select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(2173)) {
                                    select_bf16_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(28)) {
                                        select_bf16_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(139)) {
                                            select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (k < INT64_C(3259)) {
                                                select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_bf16_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                }
                            }
                        }
                    } else {
                        select_bf16_nt_config out = {4u, 1u, 4u, 16u, 16u};
                        return out;
                    }
                } else {
                    if (n < INT64_C(2509)) {
                        if (m < INT64_C(8870)) {
                            if (k < INT64_C(1537)) {
                                if (m < INT64_C(4435)) {
                                    select_bf16_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    if (n < INT64_C(182)) {
                                        select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_nt_config out = {4u, 1u, 4u, 16u, 16u};
                                        return out;
                                    }
                                }
                            } else {
                                if (k < INT64_C(2173)) {
                                    if (m < INT64_C(1268)) {
                                        select_bf16_nt_config out = {4u, 1u, 4u, 16u, 16u};
                                        return out;
                                    } else {
                                        select_bf16_nt_config out = {8u, 1u, 8u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (m < INT64_C(4435)) {
                                        if (k < INT64_C(3259)) {
                                            if (n < INT64_C(363)) {
                                                if (m < INT64_C(1109)) {
                                                    select_bf16_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    if (m < INT64_C(2218)) {
                                                        select_bf16_nt_config out = {4u, 1u, 4u, 16u, 16u};
                                                        return out;
                                                    } else {
                                                        select_bf16_nt_config out = {2u, 1u, 8u, 16u, 16u};
                                                        return out;
                                                    }
                                                }
                                            } else {
                                                if (m < INT64_C(2218)) {
                                                    select_bf16_nt_config out = {2u, 1u, 8u, 16u, 16u};
                                                    return out;
                                                } else {
                                                    select_bf16_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        } else {
                                            if (m < INT64_C(1109)) {
                                                select_bf16_nt_config out = {2u, 1u, 8u, 16u, 16u};
                                                return out;
                                            } else {
                                                select_bf16_nt_config out = {8u, 1u, 8u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    } else {
                                        if (k < INT64_C(3259)) {
                                            if (n < INT64_C(363)) {
                                                select_bf16_nt_config out = {8u, 1u, 8u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_bf16_nt_config out = {2u, 1u, 8u, 16u, 16u};
                                                return out;
                                            }
                                        } else {
                                            select_bf16_nt_config out = {8u, 1u, 8u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            }
                        } else {
                            if (n < INT64_C(182)) {
                                if (m < INT64_C(17740)) {
                                    select_bf16_nt_config out = {8u, 1u, 8u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_nt_config out = {8u, 2u, 4u, 16u, 16u};
                                    return out;
                                }
                            } else {
                                if (n < INT64_C(363)) {
                                    if (m < INT64_C(17740)) {
                                        select_bf16_nt_config out = {2u, 1u, 8u, 16u, 16u};
                                        return out;
                                    } else {
                                        select_bf16_nt_config out = {4u, 1u, 8u, 16u, 16u};
                                        return out;
                                    }
                                } else {
                                    select_bf16_nt_config out = {4u, 1u, 8u, 16u, 16u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        select_bf16_nt_config out = {4u, 1u, 8u, 16u, 16u};
                        return out;
                    }
                }
            } else {
                select_bf16_nt_config out = {8u, 1u, 8u, 8u, 8u};
                return out;
            }
        }
    } else {
        if (k < INT64_C(384)) {
            if (n < INT64_C(192)) {
                if (n < INT64_C(20)) {
                    select_bf16_nt_config out = {8u, 2u, 4u, 16u, 16u};
                    return out;
                } else {
                    if (m < INT64_C(70960)) {
                        if (k < INT64_C(42)) {
                            if (k < INT64_C(26)) {
                                select_bf16_nt_config out = {2u, 2u, 4u, 16u, 16u};
                                return out;
                            } else {
                                select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            select_bf16_nt_config out = {2u, 2u, 4u, 16u, 16u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(141920)) {
                            select_bf16_nt_config out = {8u, 2u, 4u, 16u, 16u};
                            return out;
                        } else {
                            if (k < INT64_C(63)) {
                                select_bf16_nt_config out = {2u, 2u, 4u, 16u, 16u};
                                return out;
                            } else {
                                select_bf16_nt_config out = {8u, 2u, 4u, 16u, 16u};
                                return out;
                            }
                        }
                    }
                }
            } else {
                select_bf16_nt_config out = {4u, 1u, 8u, 16u, 16u};
                return out;
            }
        } else {
            if (k < INT64_C(1630)) {
                select_bf16_nt_config out = {8u, 2u, 4u, 16u, 16u};
                return out;
            } else {
                select_bf16_nt_config out = {4u, 1u, 8u, 16u, 16u};
                return out;
            }
        }
    }
}

#endif /* SELECT_BF16_NT_H */

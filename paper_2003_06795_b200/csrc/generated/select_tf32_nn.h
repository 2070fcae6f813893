#ifndef SELECT_TF32_NN_H
#define SELECT_TF32_NN_H

#include <stdint.h>

typedef struct {
    uint32_t acc;
    uint32_t row_tile;
    uint32_t col_tile;
    uint32_t wg_rows;
    uint32_t wg_cols;
} select_tf32_nn_config;

static inline select_tf32_nn_config select_tf32_nn(int64_t m, int64_t k, int64_t n) {
    (void)m;
    (void)k;
    (void)n;
    if (m < INT64_C(17740)) {
        if (m < INT64_C(4435)) {
            if (n < INT64_C(444)) {
                if (n < INT64_C(46)) {
                    if (m < INT64_C(2218)) {
                        if (k < INT64_C(167)) {
                            select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (k < INT64_C(118)) {
                            select_tf32_nn_config out = {2u, 1u, 1u, 16u, 16u};
                            return out;
                        } else {
                            select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    }
                } else {
                    if (m < INT64_C(555)) {
                        if (k < INT64_C(157)) {
                            select_tf32_nn_config out = {2u, 1u, 1u, 16u, 16u};
                            return out;
                        } else {
                            if (n < INT64_C(287)) {
                                if (m < INT64_C(139)) {
                                    select_tf32_nn_config out = {2u, 1u, 1u, 16u, 16u};
                                    return out;
                                } else {
                                    if (k < INT64_C(1536)) {
                                        if (k < INT64_C(544)) {
                                            if (n < INT64_C(79)) {
                                                select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (m < INT64_C(317)) {
                                                    select_tf32_nn_config out = {2u, 1u, 1u, 16u, 16u};
                                                    return out;
                                                } else {
                                                    if (k < INT64_C(444)) {
                                                        select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        select_tf32_nn_config out = {2u, 1u, 1u, 16u, 16u};
                                                        return out;
                                                    }
                                                }
                                            }
                                        } else {
                                            if (k < INT64_C(992)) {
                                                if (m < INT64_C(278)) {
                                                    if (k < INT64_C(744)) {
                                                        select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                } else {
                                                    if (k < INT64_C(744)) {
                                                        if (n < INT64_C(124)) {
                                                            select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        } else {
                                                            select_tf32_nn_config out = {2u, 1u, 1u, 16u, 16u};
                                                            return out;
                                                        }
                                                    } else {
                                                        select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                }
                                            } else {
                                                if (m < INT64_C(278)) {
                                                    select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        }
                                    } else {
                                        select_tf32_nn_config out = {2u, 1u, 1u, 16u, 16u};
                                        return out;
                                    }
                                }
                            } else {
                                if (m < INT64_C(196)) {
                                    select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_nn_config out = {2u, 1u, 1u, 16u, 16u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (n < INT64_C(152)) {
                            if (k < INT64_C(222)) {
                                if (m < INT64_C(2218)) {
                                    select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(68)) {
                                        select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                if (k < INT64_C(444)) {
                                    if (n < INT64_C(111)) {
                                        if (k < INT64_C(314)) {
                                            select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (m < INT64_C(1568)) {
                                                if (n < INT64_C(79)) {
                                                    select_tf32_nn_config out = {2u, 1u, 1u, 16u, 16u};
                                                    return out;
                                                } else {
                                                    select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                select_tf32_nn_config out = {2u, 1u, 1u, 16u, 16u};
                                                return out;
                                            }
                                        }
                                    } else {
                                        select_tf32_nn_config out = {2u, 1u, 1u, 16u, 16u};
                                        return out;
                                    }
                                } else {
                                    if (m < INT64_C(1109)) {
                                        if (k < INT64_C(544)) {
                                            select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        if (k < INT64_C(544)) {
                                            if (m < INT64_C(2218)) {
                                                select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            if (n < INT64_C(79)) {
                                                select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_tf32_nn_config out = {2u, 1u, 1u, 16u, 16u};
                                                return out;
                                            }
                                        }
                                    }
                                }
                            }
                        } else {
                            if (m < INT64_C(2218)) {
                                if (k < INT64_C(544)) {
                                    if (m < INT64_C(1109)) {
                                        select_tf32_nn_config out = {2u, 1u, 1u, 16u, 16u};
                                        return out;
                                    } else {
                                        select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (m < INT64_C(1109)) {
                                        if (k < INT64_C(744)) {
                                            select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        if (k < INT64_C(1536)) {
                                            select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_nn_config out = {2u, 1u, 1u, 16u, 16u};
                                            return out;
                                        }
                                    }
                                }
                            } else {
                                if (k < INT64_C(46)) {
                                    select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(725)) {
                                        select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(1087)) {
                                            select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (k < INT64_C(1630)) {
                                                select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                }
                            }
                        }
                    }
                }
            } else {
                if (m < INT64_C(2535)) {
                    if (k < INT64_C(10752)) {
                        if (n < INT64_C(544)) {
                            if (k < INT64_C(182)) {
                                select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(363)) {
                                    select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(634)) {
                                        if (m < INT64_C(278)) {
                                            if (k < INT64_C(1449)) {
                                                if (m < INT64_C(70)) {
                                                    select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    if (m < INT64_C(139)) {
                                                        select_tf32_nn_config out = {2u, 1u, 1u, 16u, 16u};
                                                        return out;
                                                    } else {
                                                        select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                }
                                            } else {
                                                if (k < INT64_C(3072)) {
                                                    select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    if (m < INT64_C(139)) {
                                                        select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                }
                                            }
                                        } else {
                                            if (k < INT64_C(2173)) {
                                                select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_tf32_nn_config out = {2u, 1u, 1u, 16u, 16u};
                                                return out;
                                            }
                                        }
                                    } else {
                                        if (k < INT64_C(3259)) {
                                            if (m < INT64_C(1109)) {
                                                if (k < INT64_C(1449)) {
                                                    select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_nn_config out = {2u, 1u, 1u, 16u, 16u};
                                                    return out;
                                                }
                                            } else {
                                                select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            if (m < INT64_C(1109)) {
                                                select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                }
                            }
                        } else {
                            if (m < INT64_C(555)) {
                                if (n < INT64_C(1145)) {
                                    if (m < INT64_C(278)) {
                                        if (m < INT64_C(139)) {
                                            if (m < INT64_C(2)) {
                                                select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (m < INT64_C(3)) {
                                                    if (k < INT64_C(2897)) {
                                                        select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                                        return out;
                                                    }
                                                } else {
                                                    if (m < INT64_C(29)) {
                                                        if (k < INT64_C(1620)) {
                                                            if (m < INT64_C(12)) {
                                                                select_tf32_nn_config out = {2u, 1u, 1u, 16u, 16u};
                                                                return out;
                                                            } else {
                                                                select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                                return out;
                                                            }
                                                        } else {
                                                            if (m < INT64_C(12)) {
                                                                if (m < INT64_C(6)) {
                                                                    if (k < INT64_C(2897)) {
                                                                        select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                                        return out;
                                                                    } else {
                                                                        select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                                                        return out;
                                                                    }
                                                                } else {
                                                                    select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                                    return out;
                                                                }
                                                            } else {
                                                                if (k < INT64_C(2897)) {
                                                                    select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                                                    return out;
                                                                } else {
                                                                    select_tf32_nn_config out = {2u, 1u, 1u, 16u, 16u};
                                                                    return out;
                                                                }
                                                            }
                                                        }
                                                    } else {
                                                        select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                }
                                            }
                                        } else {
                                            if (k < INT64_C(124)) {
                                                select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_tf32_nn_config out = {2u, 1u, 1u, 16u, 16u};
                                                return out;
                                            }
                                        }
                                    } else {
                                        select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (m < INT64_C(70)) {
                                        if (m < INT64_C(12)) {
                                            if (m < INT64_C(3)) {
                                                select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (m < INT64_C(6)) {
                                                    select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        } else {
                                            select_tf32_nn_config out = {2u, 1u, 1u, 16u, 16u};
                                            return out;
                                        }
                                    } else {
                                        if (m < INT64_C(278)) {
                                            if (k < INT64_C(725)) {
                                                select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (m < INT64_C(139)) {
                                                    select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        } else {
                                            if (k < INT64_C(405)) {
                                                select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (k < INT64_C(725)) {
                                                    select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        }
                                    }
                                }
                            } else {
                                if (m < INT64_C(1792)) {
                                    if (k < INT64_C(124)) {
                                        if (m < INT64_C(1109)) {
                                            select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        if (m < INT64_C(896)) {
                                            if (k < INT64_C(203)) {
                                                select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (k < INT64_C(405)) {
                                                    select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    if (k < INT64_C(725)) {
                                                        select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                                        return out;
                                                    }
                                                }
                                            }
                                        } else {
                                            if (m < INT64_C(1268)) {
                                                select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                } else {
                                    select_tf32_nn_config out = {8u, 2u, 8u, 16u, 16u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (m < INT64_C(2)) {
                            select_tf32_nn_config out = {8u, 2u, 8u, 16u, 16u};
                            return out;
                        } else {
                            select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    }
                } else {
                    if (k < INT64_C(182)) {
                        select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        if (k < INT64_C(1087)) {
                            select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    }
                }
            }
        } else {
            if (k < INT64_C(1630)) {
                if (n < INT64_C(222)) {
                    if (k < INT64_C(146)) {
                        if (k < INT64_C(20)) {
                            select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (k < INT64_C(118)) {
                                if (k < INT64_C(26)) {
                                    if (m < INT64_C(8870)) {
                                        select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (m < INT64_C(8870)) {
                                    if (n < INT64_C(28)) {
                                        select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (n < INT64_C(28)) {
                                        select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            }
                        }
                    } else {
                        if (k < INT64_C(363)) {
                            if (m < INT64_C(8870)) {
                                if (k < INT64_C(222)) {
                                    select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (m < INT64_C(8870)) {
                                if (n < INT64_C(91)) {
                                    select_tf32_nn_config out = {2u, 1u, 1u, 16u, 16u};
                                    return out;
                                } else {
                                    select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                    return out;
                }
            } else {
                if (n < INT64_C(363)) {
                    if (m < INT64_C(8870)) {
                        select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        select_tf32_nn_config out = {8u, 2u, 8u, 16u, 16u};
                        return out;
                    }
                } else {
                    select_tf32_nn_config out = {8u, 2u, 8u, 16u, 16u};
                    return out;
                }
            }
        }
    } else {
        if (k < INT64_C(815)) {
            if (n < INT64_C(28)) {
                if (k < INT64_C(56)) {
                    if (m < INT64_C(35480)) {
                        select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                        return out;
                    } else {
                        select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                } else {
                    if (m < INT64_C(35480)) {
                        if (k < INT64_C(118)) {
                            select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_tf32_nn_config out = {2u, 1u, 1u, 16u, 16u};
                            return out;
                        }
                    } else {
                        select_tf32_nn_config out = {2u, 1u, 1u, 16u, 16u};
                        return out;
                    }
                }
            } else {
                if (k < INT64_C(385)) {
                    if (m < INT64_C(35480)) {
                        if (k < INT64_C(97)) {
                            select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            if (k < INT64_C(194)) {
                                select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                } else {
                    if (n < INT64_C(91)) {
                        if (m < INT64_C(50176)) {
                            select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(35480)) {
                            select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            select_tf32_nn_config out = {8u, 2u, 8u, 16u, 16u};
                            return out;
                        }
                    }
                }
            }
        } else {
            if (m < INT64_C(35480)) {
                select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                return out;
            } else {
                select_tf32_nn_config out = {8u, 2u, 8u, 16u, 16u};
                return out;
            }
        }
    }
}

#endif /* SELECT_TF32_NN_H */
